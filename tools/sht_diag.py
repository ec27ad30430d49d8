"""SHT checks at large L: exact low-degree maps through sht_forward / sht_inverse separately."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math
import numpy as np, torch
import paper_1511_05578_b200 as sc
torch.cuda.set_device(0)
for L in [int(x) for x in sys.argv[1].split(",")]:
    K = 2 * L - 1
    th = np.pi * (2 * np.arange(L) + 1) / K
    for (l, m, name, fn) in [(0, 0, "Y00", lambda t: np.full_like(t, 1 / math.sqrt(4 * math.pi))),
                             (1, 0, "Y10", lambda t: math.sqrt(3 / (4 * math.pi)) * np.cos(t)),
                             (2, 0, "Y20", lambda t: math.sqrt(5 / (16 * math.pi)) * (3 * np.cos(t) ** 2 - 1))]:
        fmap = np.repeat(fn(th)[:, None], K, axis=1).astype(np.complex128)
        fg = sc.SphereSignal(sc.SphereGrid(L), 0, torch.as_tensor(fmap, device="cuda"))
        flm = sc.sht_forward(fg).values.cpu().numpy()
        ref = np.zeros(L * L, complex); ref[l * l + l + m] = 1.0
        e_f = np.abs(flm - ref).max()
        worst = int(np.abs(flm - ref).argmax()); wl = int(math.isqrt(worst))
        inv = sc.sht_inverse(sc.HarmonicCoeffs(L, 0, torch.as_tensor(ref, device="cuda"))).values.cpu().numpy()
        e_i = np.abs(inv - fmap).max() / np.abs(fmap).max()
        print(f"L={L} {name}: forward abs err {e_f:.2e} (worst l={wl}, m={worst - wl*wl - wl}), inverse rel err {e_i:.2e}", flush=True)
