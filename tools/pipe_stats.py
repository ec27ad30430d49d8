"""Per-role cycle split of the ring kernels (build with -DSCV_PIPE_STATS=1):
runs one slab analysis + synthesis at L (default 1024) and prints the counters."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1511_05578_b200 as sc
from paper_1511_05578_b200 import _cabi
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 32
L = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
rng = np.random.default_rng(0)
w = rng.standard_normal((2, L, 2 * L - 1)) + 1j * rng.standard_normal((2, L, 2 * L - 1))
cw = sc.CurveletWignerCoeffs(L, w); grid = sc.SO3Grid(L, L, L)
lib = _cabi.load_library()
buf = (ctypes.c_ulonglong * 36)()
for it in range(2):
    torch.cuda.synchronize(); lib.scv_debug_pipe_stats(None, 1)
    slab = sc.so3_inverse_curvelet_slab(cw, grid, min(400, L - nb), nb)
    part = sc.so3_forward_curvelet_slab(slab)
    torch.cuda.synchronize(); lib.scv_debug_pipe_stats(buf, 0)
names = ["rows", "colgen", "gamma_q"]
for k in range(3):
    v = [buf[k * 6 + i] for i in range(6)]
    tw, tc, iw, idr, ifl = v[:5]
    if tc == 0: continue
    print(f"{names[k]:8s} transform groups: wait-full {100*tw/(tw+tc):5.1f}%  transform {100*tc/(tw+tc):5.1f}%   "
          f"io warps: wait-done {100*iw/(iw+idr+ifl):5.1f}%  drain {100*idr/(iw+idr+ifl):5.1f}%  fill {100*ifl/(iw+idr+ifl):5.1f}%   "
          f"(cycles/1e6: {tw/1e6:.1f} {tc/1e6:.1f} | {iw/1e6:.1f} {idr/1e6:.1f} {ifl/1e6:.1f})")
v = [buf[18 + i] for i in range(6)]
tot = sum(v) or 1
print("colgen fill split: copy issue %.1f%%  closed-form start %.1f%%  copy wait %.1f%%  scaling %.1f%%  (cycles/1e6 %s)" % (
    100 * v[0] / tot, 100 * v[1] / tot, 100 * v[2] / tot, 100 * v[3] / tot, [round(x / 1e6, 1) for x in v[:4]]))
v = [buf[24 + i] for i in range(6)]
tot = sum(v) or 1
print("gamma_q drain split: weight issue %.1f%%  wait done %.1f%%  accumulate %.1f%%  flush+barrier %.1f%%  (cycles/1e6 %s)" % (
    100 * v[0] / tot, 100 * v[1] / tot, 100 * v[2] / tot, 100 * v[3] / tot, [round(x / 1e6, 1) for x in v[:4]]))
