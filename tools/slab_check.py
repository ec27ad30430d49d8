"""K=2047 kernels on a beta slab of L=1024: one slab analysis + synthesis for
the library named by SCV_LIB; writes a digest (max, sums, sampled entries) to
gpurun_out/slab_<tag>.npz so two builds can be compared.  Random W with the
|m| <= l support of curvelet coefficients.
usage: slab_check.py TAG [b0 nb] | slab_check.py --cmp TAG1 TAG2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if sys.argv[1] == "--cmp":
    a = np.load(f"gpurun_out/slab_{sys.argv[2]}.npz")
    b = np.load(f"gpurun_out/slab_{sys.argv[3]}.npz")
    for k in a.files:
        d = np.max(np.abs(a[k] - b[k])) / max(np.max(np.abs(a[k])), 1e-300)
        print(f"{k:10s} rel diff {d:.3e}  (max {np.max(np.abs(a[k])):.3e})")
    sys.exit(0)

import torch
import paper_1511_05578_b200 as sc

tag = sys.argv[1]
L = 1024
b0 = int(sys.argv[2]) if len(sys.argv) > 2 else 500
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 8
K = 2 * L - 1
rng = np.random.default_rng(1)
w = rng.standard_normal((2, L, K)) + 1j * rng.standard_normal((2, L, K))
m = np.abs(np.arange(K) - (L - 1))[None, None, :]
l = np.arange(L)[None, :, None]
w = np.where(m <= l, w, 0.0)
w[1, 0] = 0.0
cw = sc.CurveletWignerCoeffs(L, w)
grid = sc.SO3Grid(L, L, L)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
slab = sc.so3_inverse_curvelet_slab(cw, grid, b0, nb)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0.record()
    slab = sc.so3_inverse_curvelet_slab(cw, grid, b0, nb)
    e1.record()
    torch.cuda.synchronize()
    ts.append(round(e0.elapsed_time(e1), 2))
print("analysis reps (ms):", ts)
t_ana = min(ts)
part = sc.so3_forward_curvelet_slab(slab)
torch.cuda.synchronize()
e0.record()
part = sc.so3_forward_curvelet_slab(slab)
e1.record()
torch.cuda.synchronize()
t_syn = e0.elapsed_time(e1)
v = slab.values
idx = torch.as_tensor(rng.integers(0, v.numel(), 200000), device=v.device)
samp = v.reshape(-1)[idx].cpu().numpy()
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/slab_{tag}.npz", samp=samp, sums=v.sum(dim=(0, 2)).cpu().numpy(),
         part=part.values.cpu().numpy()[:, ::37, ::5])
print(f"{tag}: analysis {t_ana:.2f} ms, synthesis {t_syn:.2f} ms for {nb} beta rows; |slab| max {float(v.abs().max()):.3e}, "
      f"nan {bool(torch.isnan(v.real).any())}")
