"""Frame-rotation kernels (csrc/rotate.cu) at one band limit: CUDA-event time
per launch and achieved HBM GB/s against MEASURED_PEAKS.json.

    python tools/rotbench.py [L=1024] [reps=5]

Algorithmic bytes: rotate_to_north writes 16 B per dense entry and reads the
(2, L, 2L-1) sparse input once; rotate_from_north reads 16 B per dense entry
and writes the sparse output.  The (L, 2L-1) edge table (33 MB at L=1024) is
L2-resident and not counted.  Inputs (22.9 GB at L=1024) exceed the 126 MB L2.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1511_05578_b200 as sc
from paper_1511_05578_b200 import _cabi

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
t = sc.build_tiling(sc.TilingParams(L, 0, 2.0, max(0, L.bit_length() - 8)))
j = t.params.j_max
g = torch.Generator(device="cuda").manual_seed(0)
v = torch.complex(torch.rand((2, L, 2 * L - 1), generator=g, device="cuda", dtype=torch.float64),
                  torch.rand((2, L, 2 * L - 1), generator=g, device="cuda", dtype=torch.float64))
ell = torch.arange(L, device="cuda")[:, None]
m = torch.arange(2 * L - 1, device="cuda")[None, :] - (L - 1)
v *= (m.abs() <= ell)[None]  # the reference's random() support: |m| <= l, no w[1, 0]
v[1, 0] = 0
w = sc.CurveletWignerCoeffs(L, v)
ctx = _cabi.context(0)
n_dense = L * (4 * L * L - 1) // 3
sparse_b = 2 * L * (2 * L - 1) * 16
peak = None
try:
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass


def timed(fn):
    for _ in range(2):
        out = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / reps


dense, t_to = timed(lambda: sc.rotate_to_north(w, j, t))
back, t_from = timed(lambda: sc.rotate_from_north(dense, j, t))
err = float((back.values - w.values).abs().max() / w.values.abs().max())
res = {"L": L, "dense_entries": n_dense, "dense_GB": n_dense * 16 / 1e9, "roundtrip_err": err}
for name, ms, by in (("rotate_to_north", t_to, n_dense * 16 + sparse_b),
                     ("rotate_from_north", t_from, n_dense * 16 + sparse_b)):
    gbs = by / ms / 1e6
    res[name] = {"ms": ms, "alg_GB": by / 1e9, "GB_s": gbs, "peak_GB_s": peak,
                 "frac": (gbs / peak) if peak else None}
print(json.dumps(res))
