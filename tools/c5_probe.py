"""Streamed round trip probe: roundtrip_streamed at (L, spin, J0) on cuda:0.

    python tools/c5_probe.py [L] [spin] [J0] [slab_GB]

Prints per-phase wall times (Delta / quadrature-table builds happen in the
first call), the round-trip error and peak memory.  For L <= 512 it also
checks bit-identity against synthesize(analyze(f)).
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1511_05578_b200 as sc  # noqa: E402
from bench import gaussian_flm  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
s = int(sys.argv[2]) if len(sys.argv) > 2 else 2
J0 = int(sys.argv[3]) if len(sys.argv) > 3 else 4
slab_gb = float(sys.argv[4]) if len(sys.argv) > 4 else 8.0
torch.cuda.set_device(0)
p = sc.TilingParams(L, s, 2.0, J0)
t = sc.build_tiling(p)
flm = gaussian_flm(L, s, 0, s == 0)
f = sc.sht_inverse(sc.HarmonicCoeffs(L, s, flm))
torch.cuda.synchronize()
nslab = [0]


def consumer(j, x):
    nslab[0] += 1


for it in range(3):
    torch.cuda.synchronize()
    t0 = time.time()
    g = sc.roundtrip_streamed(f, t, slab_bytes=int(slab_gb * (1 << 30)), consumer=consumer)
    torch.cuda.synchronize()
    dt = time.time() - t0
    err = float((g.values - f.values).abs().max() / f.values.abs().max())
    print(f"L={L} s={s} J0={J0} iter {it}: {dt:.2f} s  roundtrip rel err {err:.3e}  slabs/consumer calls {nslab[0]}  "
          f"peak {torch.cuda.max_memory_allocated() / 1e9:.1f} GB + ws {sc._cabi.context(0).workspace_bytes() / 1e9:.1f} GB",
          flush=True)
    nslab[0] = 0
if L <= 512:
    g2 = sc.synthesize(sc.analyze(f, t), t)
    print("bit-identical to synthesize(analyze(f)):", bool(torch.equal(g.values, g2.values)))
