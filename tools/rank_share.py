"""Critical path of ONE rank of the world-N sharded map, measured alone on one GPU.

The N-GPU default of bench.py shards one map (dist.analyze_sharded / synthesize_sharded:
NCCL broadcast of f_lm, beta slabs of the large scales, one NCCL reduce).  With one GPU per
call that path cannot be timed, and ranks that wait on one another must not share a GPU
(B200_PROFILING.md).  dist.VirtualRank runs a single rank's share with the two collectives
skipped, so this tool times, for N = 1, 2, 4, 8, the share of rank 0 (which also does the
SHTs, the scaling part and the final merge) and of the last rank.  1 / max over the ranks'
shares is the throughput the decomposition allows before the collectives (16.8 MB broadcast
+ 134 MB reduce at C4) -- an upper bound for the real N-GPU run, not a measurement of it.

--streamed times dist.roundtrip_sharded_streamed instead (coefficients never held: the way
BASELINE C5, L=2048 spin 2, is meant to run on 8 GPUs), with --slab-gb GiB pieces.

usage: python tools/rank_share.py [L spin jmin] [--steps K] [--worlds 1,2,4,8] [--streamed] [--slab-gb G] [--json out]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1511_05578_b200 as sc  # noqa: E402
from paper_1511_05578_b200.dist import (CudaBackend, ScalePlan, VirtualRank, analyze_sharded,  # noqa: E402
                                        roundtrip_sharded_streamed, synthesize_sharded)
from bench import gaussian_flm  # BASELINE.json's input recipe  # noqa: E402


def main():
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 3
    out = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else ""
    worlds = tuple(int(x) for x in sys.argv[sys.argv.index("--worlds") + 1].split(",")) if "--worlds" in sys.argv \
        else (1, 2, 4, 8)
    streamed = "--streamed" in sys.argv
    slab_gb = float(sys.argv[sys.argv.index("--slab-gb") + 1]) if "--slab-gb" in sys.argv else 16.0
    skip = {"--steps", "--json", "--worlds", "--slab-gb"}
    args = [x for i, x in enumerate(sys.argv[1:], 1) if not x.startswith("--") and sys.argv[i - 1] not in skip]
    L, spin, jmin = (int(args[0]), int(args[1]), int(args[2])) if len(args) >= 3 else (1024, 0, 3)
    torch.cuda.set_device(0)
    p = sc.TilingParams(L, spin, 2.0, jmin)
    t = sc.build_tiling(p)
    flm = torch.from_numpy(gaussian_flm(L, spin, 0, spin == 0)).cuda()
    f = sc.sht_inverse(sc.HarmonicCoeffs(L, spin, flm))
    be = CudaBackend()
    rows = []
    K_fin = 2 * L - 1
    slab_rows = max(1, int(slab_gb * (1 << 30)) // (K_fin * K_fin * 16))
    for world in worlds:
        plan = ScalePlan.build(p, world, True, real=False)
        for rank in sorted({0, world - 1}):
            vr = VirtualRank(rank, world)

            def step():
                if streamed:
                    return roundtrip_sharded_streamed(f, t, group=vr, backend=be, slab_rows=slab_rows)
                c = analyze_sharded(f, t, group=vr, backend=be)
                g = synthesize_sharded(c, t, group=vr, backend=be)
                del c
                return g

            for _ in range(1 if streamed else 2):
                step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                step()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            share = plan.load(rank) / sum(plan.cost)
            rows.append({"world": world, "rank": rank, "ms_per_map": ms, "volume_share": share,
                         "peak_GB": torch.cuda.max_memory_allocated() / 1e9})
            print(f"world {world} rank {rank}: {ms:8.2f} ms/map  volume share {share:.4f}", flush=True)
            be.lift_table_restrictions(plan)
            torch.cuda.empty_cache()
            torch.cuda.reset_peak_memory_stats()
    base = max((r["ms_per_map"] for r in rows if r["world"] == 1), default=None)
    summary = []
    for world in worlds:
        worst = max(r["ms_per_map"] for r in rows if r["world"] == world)
        row = {"world": world, "slowest_share_ms": worst, "maps_per_s_bound": 1e3 / worst}
        msg = f"N={world}: slowest share {worst:.2f} ms -> <= {1e3 / worst:.3f} maps/s"
        if base is not None:
            row.update(speedup_bound=base / worst, efficiency_bound=base / worst / world)
            msg += f", speed-up bound {base / worst:.2f}x ({100 * base / worst / world:.1f}% of linear)"
        summary.append(row)
        print(msg)
    if out:
        json.dump({"config": {"L": L, "spin": spin, "jmin": jmin, "steps": steps, "streamed": streamed,
                              "slab_GiB": slab_gb if streamed else None,
                              "note": "one rank's share run alone with the collectives skipped (dist.VirtualRank); "
                                      "an upper bound for the N-GPU run, not a measurement of it"},
                   "shares": rows, "summary": summary}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
