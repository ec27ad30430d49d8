"""One forward + one inverse SHT at L (default 1024) for ncu captures of the SHT kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1511_05578_b200 as sc
from bench import gaussian_flm  # BASELINE.json input recipe

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
flm = sc.HarmonicCoeffs(L, 0, gaussian_flm(L, 0, seed=0, real=True))
for _ in range(2):
    f = sc.sht_inverse(flm)
    g = sc.sht_forward(f)
torch.cuda.synchronize()
print("sht round trip", float((g.values - flm.values).abs().max() / flm.values.abs().max()))
