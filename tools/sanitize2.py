"""compute-sanitizer workload for the round-2 kernels: ring kernels at K = 1023 and 2047 on small
beta slabs, the GEMM build of the beta-quadrature table (whole and restricted to a slab)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1511_05578_b200 as sc
from paper_1511_05578_b200 import _cabi
torch.cuda.set_device(0)
ctx = _cabi.context(0)
rng = np.random.default_rng(1)
for L, b0, nb in [(512, 100, 3), (1024, 500, 2)]:
    w = np.zeros((2, L, 2 * L - 1), complex)
    for l in range(L):
        w[:, l, L - 1 - l:L + l] = rng.standard_normal((2, 2 * l + 1)) + 1j * rng.standard_normal((2, 2 * l + 1))
    cw = sc.CurveletWignerCoeffs(L, torch.as_tensor(w, device="cuda"))
    ctx.betaq_restrict(L, b0, nb)  # the table build (GEMMs) only for the slab's rows: fast under the sanitizer
    slab = sc.so3_inverse_curvelet_slab(cw, sc.SO3Grid(L, L, L), b0, nb)
    part = sc.so3_forward_curvelet_slab(slab)
    torch.cuda.synchronize()
    print(f"L={L} slab ok", float(part.values.abs().max()), flush=True)
    ctx.betaq_restrict(L, 0, 0)
    del slab, part, cw
    ctx.trim()
out = torch.empty(128 ** 3, dtype=torch.float64, device="cuda")
ctx.call("debug_betaq_build", 128, 1, _cabi.ptr(out), 128 ** 3)
torch.cuda.synchronize()
print("betaq gemm build L=128 ok", float(out.abs().max()))
print("sanitize2 workload done")
