"""compute-sanitizer workload for the SURVEY 8(f) kernels: frame rotation, SHT
wedge-pair kernels (inside a round trip), sparsity statistics (resident and
streamed), dense O(L^4) transforms, graph/lane replay."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1511_05578_b200 as sc
from paper_1511_05578_b200 import sparsity as S
from bench import gaussian_flm
torch.cuda.set_device(0)
rng = np.random.default_rng(2)
for L, s, J0 in [(32, 2, 1), (64, 0, 2)]:
    t = sc.build_tiling(sc.TilingParams(L, s, 2.0, J0))
    f = sc.sht_inverse(sc.HarmonicCoeffs(L, s, gaussian_flm(L, s, 0, s == 0)))
    c = sc.analyze(f, t)
    g = sc.synthesize(c, t)
    for j in (t.params.j_min, t.params.j_max):
        w = sc.so3_forward_curvelet(c.scale(j))
        d = sc.rotate_to_north(w, j, t)
        b = sc.rotate_from_north(d, j, t)
    summ, rows = S.sparsity_report(c, 9)
    summ2, _ = S.sparsity_report_streamed(f, t, 9)
    print(f"L={L}: rt {float((g.values - f.values).abs().max() / f.values.abs().max()):.2e}, "
          f"rot {float((b.values - w.values).abs().max()):.2e}, gini {summ['scales'][-1]['gini']:.6f}", flush=True)
dw = sc.WignerCoeffs.random(6, rng)
gr = sc.SO3Grid(8, 7, 9)
back = sc.so3_forward_general(sc.so3_inverse_general(dw, gr), 6)
print("dense", float((back.values - dw.values).abs().max()))
t = sc.build_tiling(sc.TilingParams(8, 0, 2.0, 0))
print("north", float(sc.analyze_north_validation(sc.sht_inverse(sc.HarmonicCoeffs(8, 0, gaussian_flm(8, 0, 1, True))), t, 2).values.abs().max()))
t = sc.build_tiling(sc.TilingParams(32, 0, 2.0, 2))
bt = sc.BatchedRoundTrip(t, lanes=2)
m = sc.sht_inverse(sc.HarmonicCoeffs(32, 0, gaussian_flm(32, 0, 3, True))).values
out = bt(torch.stack([m, m, m]))
torch.cuda.synchronize()
print("lanes", float((out[2] - m).abs().max()))
print("sanitize workload done")
