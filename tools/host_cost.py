"""Host time of every C-ABI stage call of an eager round trip at a small band limit
(launch-bound sizes).  usage: host_cost.py [L] [spin] [reps]"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1511_05578_b200 as sc
from paper_1511_05578_b200 import _cabi, transform as tr
from bench import gaussian_flm  # BASELINE.json input recipe

L = int(sys.argv[1]) if len(sys.argv) > 1 else 64
spin = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
t = sc.build_tiling(sc.TilingParams(L, spin, 2.0, 2))
f = sc.sht_inverse(sc.HarmonicCoeffs(L, spin, gaussian_flm(L, spin, seed=0, real=spin == 0)))
acc = collections.defaultdict(lambda: [0, 0.0, 0])
orig = _cabi.Context.call


def timed(self, name, *args):
    n0 = self.launch_count()
    t0 = time.perf_counter()
    orig(self, name, *args)
    dt = time.perf_counter() - t0
    a = acc[name + ":" + str(args[0] if name.startswith("sht") else args[1] if name in ("scale_product", "accumulate", "scaling_product", "accumulate_scaling") else args[0])]
    a[0] += 1
    a[1] += dt
    a[2] += self.launch_count() - n0


for _ in range(10):
    tr._synthesize_stages(tr._analyze_stages(f, t, True, False), t, False)
torch.cuda.synchronize()
_cabi.Context.call = timed
for _ in range(reps):
    tr._synthesize_stages(tr._analyze_stages(f, t, True, False), t, False)
    torch.cuda.synchronize()
_cabi.Context.call = orig
tot = 0.0
for k, (n, s, l) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:34s} calls/map {n / reps:5.1f}  host us/call {1e6 * s / n:7.1f}  launches/call {l / n:5.1f}")
    tot += s
print(f"total host time in C calls: {1e3 * tot / reps:.3f} ms per round trip")
