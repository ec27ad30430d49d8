"""SHT round trip vs L and degree band (locates the failing regime)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1511_05578_b200 as sc
torch.cuda.set_device(0)
for L in [int(x) for x in sys.argv[1].split(",")]:
    rng = np.random.default_rng(0)
    ell = np.floor(np.sqrt(np.arange(L * L))).astype(int)
    m = np.arange(L * L) - ell * ell - ell
    for lo, hi, mmax in [(0, L, L), (0, L // 2, L), (L // 2, L, L), (0, L, 64), (L - 64, L, L)]:
        v = rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)
        v[(ell < lo) | (ell >= hi) | (np.abs(m) >= mmax)] = 0
        flm = torch.as_tensor(v, device="cuda")
        f = sc.sht_inverse(sc.HarmonicCoeffs(L, 0, flm))
        back = sc.sht_forward(f).values
        err = (back - flm).abs()
        w = int(err.argmax()); wl = int(np.sqrt(w))
        print(f"L={L} l in [{lo},{hi}) |m|<{mmax}: round trip {float(err.max() / flm.abs().max()):.2e} worst l={wl} m={w - wl*wl - wl}", flush=True)
