"""Sparsity report at C4 (L=1024, J0=3) on one B200, streamed (no resident
coefficients): wall time of the whole report and of the per-scale statistics
of the finest scale (|c| pass, histogram, radix sort, Gini reduction).

    python tools/sparsitybench.py [L=1024] [bins=10]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1511_05578_b200 as sc
from bench import gaussian_flm  # BASELINE.json input recipe
from paper_1511_05578_b200 import _cabi
from paper_1511_05578_b200 import sparsity as S

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
bins = int(sys.argv[2]) if len(sys.argv) > 2 else 10
t = sc.build_tiling(sc.TilingParams(L, 0, 2.0, 3 if L >= 1024 else 2))
flm = sc.HarmonicCoeffs(L, 0, gaussian_flm(L, 0, seed=0, real=True))
f = sc.sht_inverse(flm)
S.sparsity_report_streamed(f, t, bins)  # warm-up: tables, plans
torch.cuda.synchronize()
ctx = _cabi.context(0)
ctx.profile_report()
ctx.profile(True)
t0 = time.perf_counter()
summary, rows = S.sparsity_report_streamed(f, t, bins)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
ctx.profile(False)
prof = ctx.profile_report()
n_fin = summary["scales"][-1]["coefficients"]
sp = prof.get("sparsity", (0, 0.0))
res = {"L": L, "bins": bins, "wall_s": wall, "stages_ms": {k: round(v[1], 2) for k, v in prof.items()},
       "finest_scale_coefficients": n_fin, "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9,
       "scales": summary["scales"]}
print(json.dumps(res))
