"""Repeat the L=1024 analysis SO(3) transform (gamma-first: colgen + rows) and
time each launch group with CUDA events, to see run-to-run variance."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1511_05578_b200 as sc
from paper_1511_05578_b200 import _cabi
L = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
rng = np.random.default_rng(0)
vals = rng.standard_normal((2, L, 2 * L - 1)) + 1j * rng.standard_normal((2, L, 2 * L - 1))
if len(sys.argv) > 3:  # scale degree l by (l+1)^-p, like the curvelet coefficients of a C_l=(l+1)^-2 map
    vals *= (np.arange(L) + 1.0)[None, :, None] ** -float(sys.argv[3])
w = sc.CurveletWignerCoeffs(L, vals)
grid = sc.SO3Grid(L, L, L)
K = 2 * L - 1
out = torch.empty((K, L, K), dtype=torch.complex128, device="cuda")
ctx = _cabi.context(0)
sc.so3_inverse_curvelet(w, grid, out=out)
torch.cuda.synchronize()
for i in range(reps):
    ctx.profile_report(); ctx.profile(True)
    sc.so3_inverse_curvelet(w, grid, out=out)
    ctx.profile(False)
    rep = ctx.profile_report()
    print(i, {k: round(v[1], 2) for k, v in rep.items()}, flush=True)
