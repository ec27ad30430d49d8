"""Beta-quadrature table: the tensor-core GEMM build (method 1) against the
direct sums (method 0) at band limit L -- max relative difference over the
whole table, and both build times.  usage: betaq_check.py [L ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1511_05578_b200 import _cabi

ctx = _cabi.context(0)
for L in [int(a) for a in sys.argv[1:]] or [128, 512, 1024]:
    n = L ** 3
    tabs, ts = [], []
    for method in (0, 1):
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.call("debug_betaq_build", L, method, _cabi.ptr(out), n)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        tabs.append(out)
    d = (tabs[0] - tabs[1]).abs().max().item()
    mx = tabs[0].abs().max().item()
    # per-row scale: the weights span many orders of magnitude, so also compare relative to each
    # value where it is not tiny
    big = tabs[0].abs() > 1e-6 * mx
    rel = ((tabs[0] - tabs[1]).abs()[big] / tabs[0].abs()[big]).max().item()
    print(f"L={L}: direct {ts[0]*1e3:.1f} ms, gemm {ts[1]*1e3:.1f} ms; max|diff|/max|q| = {d/mx:.3e}, "
          f"max rel diff (|q| > 1e-6 max) = {rel:.3e}, nan {bool(torch.isnan(tabs[1]).any())}", flush=True)
    del tabs, out
    torch.cuda.empty_cache()
