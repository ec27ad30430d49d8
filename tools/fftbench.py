"""Batched odd-length DFT: hand-written prime-factor engine vs cuFFT (torch.fft)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1511_05578_b200 import _cabi
ctx = _cabi.context(0)
torch.manual_seed(0)
for K in [int(k) for k in (sys.argv[1].split(",") if len(sys.argv) > 1 else "3,7,15,31,63,255,511,1023,2047,4095".split(","))]:
    n = max(1, (1 << 27) // (K * 16))  # ~128 MB per batch
    x = torch.randn(n, K, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    for d in (-1, 1):
        ctx.call("debug_dft", K, d, n, _cabi.ptr(x), _cabi.ptr(y))
        ref = torch.fft.fft(x, dim=1) if d < 0 else torch.fft.ifft(x, dim=1) * K
        err = float((y - ref).abs().max() / ref.abs().max())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            ctx.call("debug_dft", K, d, n, _cabi.ptr(x), _cabi.ptr(y))
        e1.record(); torch.cuda.synchronize()
        t_pfa = e0.elapsed_time(e1) / 5
        e0.record()
        for _ in range(5):
            torch.fft.fft(x, dim=1, out=y)
        e1.record(); torch.cuda.synchronize()
        t_cu = e0.elapsed_time(e1) / 5
        pts = n * K
        print(f"K={K:5d} dir={d:+d} rows={n:7d} err={err:.2e}  pfa {t_pfa:7.3f} ms ({pts/t_pfa/1e6:8.2f} Gpt/s)  cufft {t_cu:7.3f} ms ({pts/t_cu/1e6:8.2f} Gpt/s)", flush=True)
