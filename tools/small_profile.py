"""Host-side profile of the eager round trip at a small band limit (launch-bound sizes):
cProfile over `reps` analyze+synthesize calls.  usage: small_profile.py [L] [reps]"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1511_05578_b200 as sc
from bench import gaussian_flm  # BASELINE.json input recipe

L = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
t = sc.build_tiling(sc.TilingParams(L, 0, 2.0, 2))
f = sc.sht_inverse(sc.HarmonicCoeffs(L, 0, gaussian_flm(L, 0, seed=0, real=True)))
for _ in range(20):
    g = sc.synthesize(sc.analyze(f, t), t)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    g = sc.synthesize(sc.analyze(f, t), t)
torch.cuda.synchronize()
print(f"L={L}: {(time.perf_counter() - t0) / reps * 1e3:.3f} ms per round trip (wall, {reps} reps)")
pr = cProfile.Profile()
pr.enable()
for _ in range(reps):
    g = sc.synthesize(sc.analyze(f, t), t)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
