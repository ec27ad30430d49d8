import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1511_05578_b200 as sc
from oracle import scurve_oracle as orc
h = lambda t: t.cpu().numpy()
for L, s in [(4, 0), (8, 0), (8, 2), (32, 2)]:
    flm = orc.gaussian_flm(L, s, 0, False)
    f = sc.sht_inverse(sc.HarmonicCoeffs(L, s, flm))
    ref = orc.sht_inverse(flm, L, s)
    print("sht_inv", L, s, orc.rel_err(h(f.values), ref))
    b = sc.sht_forward(sc.SphereSignal(sc.SphereGrid(L), s, ref))
    print("sht_fwd", L, s, orc.rel_err(h(b.values), orc.sht_forward(ref, L, s)))
    rng = np.random.default_rng(0)
    w = np.zeros((2, L, 2*L-1), complex); c = L-1
    for l in range(L):
        for sh in range(2 if l else 1):
            w[sh, l, c-l:c+l+1] = rng.standard_normal(2*l+1) + 1j*rng.standard_normal(2*l+1)
    F = sc.so3_inverse_curvelet(sc.CurveletWignerCoeffs(L, w), sc.SO3Grid(L, L, L))
    Fr = orc.so3_inverse_curvelet(w)
    print("so3_inv", L, orc.rel_err(h(F.values), Fr), np.isnan(h(F.values)).sum())
    W = sc.so3_forward_curvelet(sc.SO3Signal(sc.SO3Grid(L, L, L), Fr))
    Wr = orc.so3_forward_curvelet(Fr)
    hw = h(W.values)
    print("so3_fwd", L, orc.rel_err(hw, Wr), np.isnan(hw).sum())
    if L <= 8:
        np.set_printoptions(precision=3, linewidth=200)
        print(np.abs(hw - Wr)[0]); print(np.abs(hw-Wr)[1])
