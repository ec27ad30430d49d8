"""Component checks at L = 2048 (BASELINE C5) on cuda:0:
SHT round trip, the K = 4095 DFT engine against torch.fft, and the beta-slab
SO(3) pair forward(inverse(w)) == w per scale band limit."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1511_05578_b200 as sc  # noqa: E402
from paper_1511_05578_b200 import _cabi  # noqa: E402
from bench import gaussian_flm  # noqa: E402

torch.cuda.set_device(0)
ctx = _cabi.context(0)
Ls = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1024, 2048]

for K in (2047, 4095):
    x = torch.randn(64, K, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    for d in (-1, 1):
        ctx.call("debug_dft", K, d, 64, _cabi.ptr(x), _cabi.ptr(y))
        ref = torch.fft.fft(x, dim=1) if d < 0 else torch.fft.ifft(x, dim=1) * K
        print(f"DFT K={K} dir={d:+d} rel err {float((y - ref).abs().max() / ref.abs().max()):.2e}", flush=True)

for L in Ls:
    for s in (0, 2):
        flm = torch.as_tensor(gaussian_flm(L, s, 1, False), device="cuda")
        t0 = time.time()
        f = sc.sht_inverse(sc.HarmonicCoeffs(L, s, flm))
        back = sc.sht_forward(f)
        torch.cuda.synchronize()
        print(f"SHT L={L} s={s}: round trip rel err {float((back.values - flm).abs().max() / flm.abs().max()):.2e} "
              f"({time.time() - t0:.1f} s)", flush=True)

for L in Ls:
    K = 2 * L - 1
    g = torch.Generator().manual_seed(L)
    w = torch.zeros(2, L, K, dtype=torch.complex128)
    for l in range(1, L):
        n = 2 * l + 1
        w[:, l, L - 1 - l:L + l] = torch.complex(torch.randn(2, n, generator=g, dtype=torch.float64),
                                                 torch.randn(2, n, generator=g, dtype=torch.float64))
    w = w.cuda()
    W = sc.CurveletWignerCoeffs(L, w)
    grid = sc.SO3Grid(L, L, L)
    nb = max(1, min(L, (4 << 30) // (K * K * 16)))
    acc = None
    t0 = time.time()
    for b0 in range(0, L, nb):
        nbb = min(nb, L - b0)
        slab = sc.so3_inverse_curvelet_slab(W, grid, b0, nbb)
        if acc is None:
            acc = sc.so3_forward_curvelet_slab(slab)
        else:
            sc.so3_forward_curvelet_slab(slab, out=acc.values, accumulate=True)
        del slab
    torch.cuda.synchronize()
    err = (acc.values - w).abs()
    e = float(err.max() / w.abs().max())
    li, mi = np.unravel_index(int(err[0].argmax()), err[0].shape)
    print(f"SO3 slab pair L={L}: forward(inverse(w)) rel err {e:.2e} (worst sheet-0 entry l={li}, m={mi - (L - 1)}) "
          f"({time.time() - t0:.1f} s)", flush=True)
    # error profile over l
    el = err.amax(dim=(0, 2)).cpu().numpy()
    print("  max err by l decile:", [f"{el[i * L // 10:(i + 1) * L // 10].max():.1e}" for i in range(10)], flush=True)
