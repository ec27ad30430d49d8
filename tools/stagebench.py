"""Time the K-point row engine (debug_dft -> k_pfa_rows_g) for the current
SCV_LIB variant: rows/s and G points/s (timing experiments; variants built
with SCV_EXP_* macros compute wrong results on purpose)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1511_05578_b200 import _cabi
ctx = _cabi.context(0)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 2047
nrows = int(sys.argv[2]) if len(sys.argv) > 2 else 2047 * 64
x = torch.randn(nrows, K, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
for d in (-1, 1):
    for _ in range(2):
        ctx.call("debug_dft", K, d, nrows, _cabi.ptr(x), _cabi.ptr(y))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        ctx.call("debug_dft", K, d, nrows, _cabi.ptr(x), _cabi.ptr(y))
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{os.path.basename(os.environ.get('SCV_LIB', 'base'))} K={K} dir={d:+d} rows={nrows} {ms:8.3f} ms "
          f"{nrows * K / ms / 1e6:7.2f} Gpt/s  ns/row/SM={ms * 1e6 * 148 / nrows:7.1f}", flush=True)
