"""Benchmark: curvelet analysis + synthesis maps/s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--L 1024 --spin 0 --jmin 3 --lam 2] [--real]

Default workload = BASELINE configs[3] (C4): L=1024, spin 0, B=lambda=2,
J_min=3, one map with seeded Gaussian f_lm (C_l=(l+1)^-2, real-signal
symmetry), complex128 path (analyze + synthesize).  A "step" is one full
analysis + synthesis of one map; `value` is maps/s with the input map
resident in HBM; `e2e` repeats the step through the public API with the
map copied host->device and the reconstruction copied back every step.
Every scale volume (68.6 GB at the finest scale) is far larger than the
126 MB L2, so no explicit L2 flush is needed between steps.

Multi-GPU (one process per GPU).  `--gpus N` under torchrun (WORLD_SIZE set)
uses the launched ranks; without WORLD_SIZE, bench.py launches the N ranks
itself (torch.distributed.run on 127.0.0.1) and asserts world == N.  The
N > 1 default is the north star's decomposition of ONE C4 map per step
(dist.py): rank 0 runs the SHT and NCCL-broadcasts f_lm, the scales with
128 <= L_j <= 2048 are split into one beta slab per rank, small scales are
whole per rank, and one NCCL reduce merges the per-scale synthesis terms --
strong scaling, max-over-ranks device time.  `--maps-per-rank` instead runs
one independent map per rank (weak scaling, no collective).

--impl reference times the reference algorithm's CPU implementation (the
oracle port in oracle/, numpy + scipy.fft with all host threads) on a
bounded sample of the same workload, on rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--L", type=int, default=1024)
    ap.add_argument("--spin", type=int, default=0)
    ap.add_argument("--jmin", type=int, default=3)
    ap.add_argument("--lam", type=float, default=2.0)
    ap.add_argument("--real", action="store_true", help="analyze_real/synthesize_real path")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--lanes", type=int, default=0,
                    help="N > 0: a step is a batch of N maps in flight at once (BatchedRoundTrip: N graph "
                         "lanes with private contexts and streams); small L")
    ap.add_argument("--graph", action="store_true",
                    help="replay analyze+synthesize from one captured CUDA graph (GraphedRoundTrip; "
                         "launch-bound small L)")
    ap.add_argument("--profile-json", default="")
    ap.add_argument("--streamed", action="store_true",
                    help="roundtrip_streamed: beta-slab streamed analysis+synthesis (coefficients never "
                         "held whole; BASELINE C5 on one GPU: --L 2048 --spin 2 --jmin 4)")
    ap.add_argument("--slab-gb", type=float, default=16.0, help="--streamed slab size (GiB)")
    ap.add_argument("--shard-scales", action="store_true",
                    help="(default for N>1) one map per step with its scales / beta slabs sharded over the ranks")
    ap.add_argument("--maps-per-rank", action="store_true",
                    help="N>1: one independent map per rank per step (weak scaling, no collective)")
    ap.add_argument("--stub", action="store_true",
                    help="launcher / collective plumbing check on CPU (gloo, no transform compute); tests only")
    ap.add_argument("--no-measured-cpu", action="store_true",
                    help="skip the measured full CPU round trip at L=256 (cpu_baseline.measured)")
    return ap.parse_args()


def spawn_ranks(a) -> int:
    """`--gpus N` without WORLD_SIZE: launch N ranks of this script with
    torch.distributed.run on 127.0.0.1 and return its exit code (rank 0
    prints the JSON line)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


class _Batch:
    """A (B, L, 2L-1) batch handed to the batched step."""

    def __init__(self, values):
        self.values = values


def gaussian_flm(L, spin, seed, real):
    """BASELINE.json input recipe: Re/Im iid N(0, C_l/2)."""
    rng = np.random.default_rng(seed)
    ell = np.floor(np.sqrt(np.arange(L * L))).astype(np.int64)
    v = (rng.standard_normal(L * L) + 1j * rng.standard_normal(L * L)) * np.sqrt((ell + 1.0) ** -2 / 2.0)
    v[: spin * spin] = 0.0
    if real:
        for l in range(L):
            row = v[l * l:(l + 1) ** 2]
            row[l] = row[l].real
            ms = np.arange(1, l + 1)
            row[l - ms] = np.where(ms % 2 == 0, 1.0, -1.0) * np.conj(row[l + ms])
    return v


def workload_name(a):
    path = "analyze_real+synthesize_real" if a.real else "analyze+synthesize"
    if a.streamed:
        path = "roundtrip_streamed (beta-slab streamed analyze+synthesize)"
    return f"curvelet {path} L={a.L} spin={a.spin} B={a.lam:g} J0={a.jmin}"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons, pw = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def algorithmic_work(a):
    """Per-map algorithmic bytes / flops and per-scale sizes."""
    from paper_1511_05578_b200 import TilingParams, scale_band_limit
    p = TilingParams(a.L, a.spin, a.lam, a.jmin)
    b = 8 if a.real else 16
    Ljs = [scale_band_limit(p, j) for j in range(p.j_min, p.j_max + 1)]
    V = [(2 * Lj - 1) ** 2 * Lj for Lj in Ljs]
    B_alg = sum(2 * v * b for v in V) + 2 * a.L * (2 * a.L - 1) * b + 16 * a.L * a.L
    F_alg = sum(2 * 5 * (2 * Lj - 1) ** 3 * math.log2((2 * Lj - 1) ** 3) for Lj in Ljs)
    if a.real:
        F_alg /= 2
    return p, Ljs, B_alg, F_alg


def ncu_traffic(stage, Ljs):
    """Measured DRAM bytes (read + write) per map for `stage`, from the committed
    ncu --set full captures (profiles/ncu_traffic.json: bytes per beta row of
    the L_j = 1024 kernel on a 16-row slab, tools/prof_slab.py), scaled to the
    map's L_j = 1024 scales; None when the stage or size has no capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tab = json.load(fh)
    except Exception:
        return None
    e = tab.get(stage)
    if not e:
        return None
    n = sum(1 for L in Ljs if L == e["L"])
    if n == 0:
        return None
    return {"bytes_per_map": e["bytes_per_beta_row"] * e["L"] * n, "covers": f"{n} L_j={e['L']} scale launch(es)",
            "kernel": e["kernel"], "source": e["source"]}


# Prime-factor plans and launch shapes of the DFT engine (csrc/pfa.cuh PfaPlan,
# pfa.cu PfaCfg / PfaSCfg / PfaGCfg / PfaQCfg), mirrored to count the FP64
# tensor-core (DMMA m8n8k4, 512 flops each) instructions a pass executes:
# per call of R rows, a DMMA radix p (h = (p-1)/2) runs 2*ceil(R*(K/p)/8)
# warp blocks x ceil((h+1)/8) m8 tiles x ceil(h/4) k-steps x 2 (C.s, S.d).
# Cross-checked against ncu: 1081 DMMA per K=2047 row (sm__inst_executed_pipe_
# tensor_subpipe_dmma, profiles/r01v8_ncu_k_pfa_rows.txt) vs 1080 here with the
# dense radix-89 stage; the Rader radix-89 stage (r01v15+) issues 66 per block
# of 4 butterflies: 288 + 396 = 684 per K=2047 row.
PFA_PLAN = {3: (3,), 7: (7,), 15: (3, 5), 31: (31,), 63: (7, 9), 255: (3, 5, 17), 511: (7, 73),
            1023: (31, 33), 2047: (23, 89), 4095: (9, 13, 35)}
PFA_R = {  # rows per transform call by stage
    # (the ring kernels of K = 2047, 1023 and the K = 511 row / gamma passes transform one row per call)
    "so3inv_rows": {255: 8},
    "so3inv_colgen": {511: 4, 255: 8, 4095: 2},
    "so3fwd_alpha": {255: 8},
    "so3fwd_gamma_q": {},
}
DMMA_PEAK_TF = 36.9  # measured, 8 independent chains x 32 warps/SM (profiles/r01_fp64_pipe_microbench.log)


def dmma_per_row(K, R):
    if K not in PFA_PLAN:
        return None
    tot = 0
    for p in PFA_PLAN[K]:
        if p < (9 if K == 4095 else 17):
            continue
        h = (p - 1) // 2
        nblk = 2 * ((R * (K // p) + 7) // 8)
        if p == 89:  # Rader + 4 x 11 CRT (pfa_stage_rader89): 2*6 + 3*18 DMMA per block
            tot += nblk * 66
            continue
        tot += nblk * ((h + 1 + 7) // 8) * ((h + 3) // 4) * 2
    return tot / R


def executed_dmma(stage, Ljs):
    """Executed DMMA flops of one map's launches of `stage` (None if a scale is not on the engine)."""
    if stage not in PFA_R:
        return None
    fl = 0.0
    for L in Ljs:
        K = 2 * L - 1
        d = dmma_per_row(K, PFA_R[stage].get(K, 1))
        if d is None:
            continue
        fl += d * 512.0 * K * L  # K*L transforms of length K per pass
    return fl


def stage_roofline(a, prof, Ljs, hbm_peak, fp64_peak, dmma_peak=None):
    """Roofline of the dominant stage from the live per-stage CUDA-event times."""
    K = lambda L: 2 * L - 1  # noqa: E731
    b = 8 if a.real else 16
    # algorithmic bytes per call summed over the scales of one map (one call per scale)
    vol = sum(K(L) ** 2 * L for L in Ljs)
    cols = sum((2 * L * L - 1) * L for L in Ljs)
    bytes_stage = {
        "so3inv_alpha": 16 * vol,                     # generated in shared memory, written once
        "so3inv_gamma": 2 * 16 * vol,                 # read + write in place
        "so3inv_colgen": 16 * vol,                    # gamma-first: generated columns, written once
        "so3inv_rows": 2 * 16 * vol,                  # alpha rows read + written in place
        "so3fwd_alpha": (b + 16) * vol,               # read the scale signal + write the chunk
        "so3fwd_gamma": 16 * vol + 16 * cols,         # read the chunk + write the pruned columns
        "beta_so3": 16 * cols,                        # read pruned columns once
        # gamma pass fused with the beta quadrature: read the chunk + one table double per (n, m, b)
        "so3fwd_gamma_q": 16 * vol + 8 * cols,
    }
    def P_of(L):
        return 1 << max(4, math.ceil(math.log2(4 * L - 3)))
    # algorithmic FP64 flops (5 N log2 N per complex transform):
    #   alpha/gamma passes: one K-point transform per row / column of the volume
    #   beta stage: the paper's per-column work -- one K-point DFT + the padded
    #   weight convolution (two P-point transforms) -- for the 2L^2-1 columns
    flops_stage = {
        "so3inv_alpha": sum(K(L) * L * 5 * K(L) * math.log2(K(L)) for L in Ljs),
        "so3inv_gamma": sum(K(L) * L * 5 * K(L) * math.log2(K(L)) for L in Ljs),
        "so3inv_colgen": sum(K(L) * L * 5 * K(L) * math.log2(K(L)) for L in Ljs),
        "so3inv_rows": sum(K(L) * L * 5 * K(L) * math.log2(K(L)) for L in Ljs),
        "so3fwd_alpha": sum(K(L) * L * 5 * K(L) * math.log2(K(L)) for L in Ljs),
        "so3fwd_gamma": sum(K(L) * L * 5 * K(L) * math.log2(K(L)) for L in Ljs),
        "beta_so3": sum((2 * L * L - 1) * (5 * K(L) * math.log2(K(L)) + 2 * 5 * P_of(L) * math.log2(P_of(L)))
                        for L in Ljs),
        # gamma transforms + 2 flops (complex x real FMA pair = 4) per (n, m, b) quadrature term
        "so3fwd_gamma_q": sum(K(L) * L * 5 * K(L) * math.log2(K(L)) + 4 * (2 * L * L - 1) * L for L in Ljs),
    }
    # per map: work of the stage over all its launches / its device time per map
    name, (cnt, ms) = max(prof.items(), key=lambda kv: kv[1][1])
    ms_map = ms / a.steps
    out = {"stage": name, "launches_per_map": cnt / a.steps, "ms_per_map": ms_map}
    if name == "beta_so3":
        ach = flops_stage[name] / (ms_map * 1e-3) / 1e12
        out.update({"bound": "fp64", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
                    "frac": ach / fp64_peak, "peak_source": "measured DFMA loop in this run (scv_fp64_peak)",
                    "hbm_gbs_alg": bytes_stage[name] / (ms_map * 1e-3) / 1e9})
    else:
        ach = bytes_stage.get(name, 0) / (ms_map * 1e-3) / 1e9
        out.update({"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                    "frac": ach / hbm_peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs"})
        if name in flops_stage:
            out["fp64_tflops_alg"] = flops_stage[name] / (ms_map * 1e-3) / 1e12
    ex = executed_dmma(name, Ljs)
    if ex:
        # what the kernel's own pipe does: FP64 tensor-core (DMMA) flops the
        # prime-factor engine issues, vs the measured DMMA peak
        pk = dmma_peak or DMMA_PEAK_TF
        out["executed_dmma"] = {"tflops": ex / (ms_map * 1e-3) / 1e12, "peak_tflops": pk,
                                "peak_source": "in-run DMMA loop (scv_dmma_peak)" if dmma_peak else "r01 microbench",
                                "frac": ex / (ms_map * 1e-3) / 1e12 / pk,
                                "flops_per_map": ex, "source": "DMMA count of the engine's launch shapes "
                                "(bench.py dmma_per_row; 684/row at K=2047 with the Rader radix-89 stage)"}
    tr = ncu_traffic(name, Ljs)
    # measured DRAM bytes (GB per map) vs the algorithmic bytes behind `achieved`
    out["traffic"] = None if tr is None else tr["bytes_per_map"] / 1e9
    out["traffic_detail"] = tr
    out["alg_GB_per_map"] = bytes_stage.get(name, 0) / 1e9
    out["all_stages"] = {}
    for nm, (c_, ms_) in prof.items():
        mm = ms_ / a.steps
        e = {"ms_per_map": mm}
        if nm in bytes_stage:
            e["hbm_gbs_alg"] = bytes_stage[nm] / (mm * 1e-3) / 1e9
        if nm in flops_stage:
            e["fp64_tflops_alg"] = flops_stage[nm] / (mm * 1e-3) / 1e12
        exn = executed_dmma(nm, Ljs)
        if exn:
            e["dmma_frac"] = exn / (mm * 1e-3) / 1e12 / (dmma_peak or DMMA_PEAK_TF)
        out["all_stages"][nm] = e
    return out


def run_stub(a):
    """--stub: the launcher and collective plumbing of the N-rank bench on CPU
    (gloo), without any transform compute -- for tests/test_bench_launcher.py.
    The line carries "stub": true and no throughput claim."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"world size {world} != --gpus {a.gpus}")
    if world > 1:
        dist.init_process_group("gloo")
    from paper_1511_05578_b200.dist import ScalePlan
    from paper_1511_05578_b200.tiling import TilingParams
    p = TilingParams(a.L, a.spin, a.lam, a.jmin)
    plan = ScalePlan.build(p, world)
    flm = torch.zeros(a.L * a.L, dtype=torch.complex128)
    terms = torch.zeros((p.scale_count, a.L * a.L), dtype=torch.complex128)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        if world > 1:
            dist.broadcast(flm, src=0)
            dist.reduce(terms, dst=0, op=dist.ReduceOp.SUM)
    el = time.perf_counter() - t0
    line = {"metric": "curvelet analysis+synthesis maps/s", "value": None, "unit": "maps/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "stub": True, "scaling": "strong",
            "config": {"workload": workload_name(a), "parallelism": f"scales + beta slabs sharded x{world}",
                       "rank_loads": [plan.load(r) for r in range(world)]},
            "collective_wall_s": el}
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def arm_config(a, p, Ljs, world, sharded, maps_per_step):
    """`config` of the JSON line; both arms print the same dict for the same flags."""
    coeff_mb = sum((2 * Lj - 1) ** 2 * Lj for Lj in Ljs) * 16 / 1e6
    return {"workload": workload_name(a), "L": a.L, "spin": a.spin, "lambda": a.lam,
            "j_min": a.jmin, "j_max": p.j_max, "scale_band_limits": Ljs,
            "maps_per_step": maps_per_step,
            **({"streamed_slab_GiB": a.slab_gb} if a.streamed else {}),
            "parallelism": ("scales + beta slabs sharded x%d%s (NCCL broadcast f_lm + reduce of the "
                            "per-scale terms)" % (world, ", slabs streamed" if a.streamed else "")
                            if sharded else
                            (f"maps x{world} (one map per rank)" if world > 1 else "1 GPU")),
            **({"cuda_graph": True} if a.graph else {}),
            **({"lanes": a.lanes, "batch": "maps in flight per step, one CUDA graph + private "
                "context + stream per lane"} if a.lanes else {}),
            "l2_flush": ("not needed: the %.0f MB of coefficients per step exceed the 126 MB L2" % coeff_mb
                         if coeff_mb > 126 else
                         "none: the %.0f MB of coefficients fit in the 126 MB L2 at this size "
                         "(small, launch-bound config)" % coeff_mb)}


def measured_cpu_roundtrip(a, gpu_ms_at):
    """cpu_baseline.measured: one FULL oracle round trip (analyze + synthesize,
    transform.py:139-187 restated) at L=256 with the bench's lambda / J0, timed
    on this host with all cores and with one scipy.fft worker, beside the GPU
    time of the same round trip (the largest L the reference
    finishes in reasonable time; L=1024 does not fit host RAM)."""
    from scipy import fft as sfft
    from oracle import scurve_oracle as orc
    from paper_1511_05578_b200 import tiling as T
    L = 256
    p = T.TilingParams(L, a.spin, a.lam, a.jmin)
    t = T.build_tiling(p)
    psi = [T.curvelet_harmonics(t, j) for j in range(p.j_min, p.j_max + 1)]
    flm = gaussian_flm(L, a.spin, a.seed, a.spin == 0)
    f = orc.sht_inverse(flm, L, a.spin)
    out = {"L": L, "config": f"L={L} spin={a.spin} B={a.lam:g} J0={a.jmin}, analyze+synthesize (complex path)"}
    for tag, workers in (("all_cores", os.cpu_count() or 1), ("one_thread", 1)):
        with sfft.set_workers(workers):
            t0 = time.perf_counter()
            smap, scales = orc.analyze(f, L, a.spin, a.lam, a.jmin, p.j_max, psi, t.scaling)
            g = orc.synthesize(smap, scales, L, a.spin, a.lam, a.jmin, p.j_max, psi, t.scaling)
            sec = time.perf_counter() - t0
        out[tag] = {"cores": workers, "s_per_map": sec}
        del smap, scales
    out["roundtrip_rel_err"] = orc.rel_err(g, f)
    out["gpu_s_per_map"] = gpu_ms_at(L) / 1e3
    out["ratio_all_cores"] = out["all_cores"]["s_per_map"] / out["gpu_s_per_map"]
    out["ratio_one_thread"] = out["one_thread"]["s_per_map"] / out["gpu_s_per_map"]
    return out


def run_ours(a):
    if a.stub:
        return run_stub(a)
    import torch
    import torch.distributed as dist

    import paper_1511_05578_b200 as sc
    from paper_1511_05578_b200 import _cabi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"world size {world} != --gpus {a.gpus} (launch with torchrun, or without WORLD_SIZE "
                         f"and bench.py spawns the ranks)")
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL prints its communicator-init lines (rank, nranks, device, NVLS)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sharded = world > 1 and not a.maps_per_rank
    dev = torch.device("cuda", local)
    t_first0 = time.perf_counter()
    ctx = _cabi.context(local)

    p, Ljs, B_alg, F_alg = algorithmic_work(a)
    t = sc.build_tiling(p)
    real_sym = a.spin == 0
    flm = gaussian_flm(a.L, a.spin, a.seed + (0 if sharded else rank), real_sym)
    f = sc.sht_inverse(sc.HarmonicCoeffs(a.L, a.spin, flm))
    if a.real:
        f = sc.SphereSignal(f.grid, 0, f.values.real.contiguous(), real=True)
    dtype = torch.float64 if a.real else torch.complex128
    ana = sc.analyze_real if a.real else sc.analyze
    syn = sc.synthesize_real if a.real else sc.synthesize
    if a.streamed:
        if a.real:
            raise SystemExit("--streamed runs the complex path")

        def step(fin):
            return sc.roundtrip_streamed(fin, t, slab_bytes=int(a.slab_gb * (1 << 30)))
    elif not sharded:
        scale_out = [torch.empty((2 * Lj - 1, Lj, 2 * Lj - 1), dtype=dtype, device=dev) for Lj in Ljs]

        def step(fin):
            c = ana(fin, t, scale_out=scale_out)
            return syn(c, t)

    eager_step = step if not sharded else None
    graphed = None
    if a.graph:
        if a.streamed or sharded:
            raise SystemExit("--graph replays the single-GPU in-memory round trip")
        graphed = sc.GraphedRoundTrip(t, spin=a.spin, real=a.real)

        def step(fin):  # noqa: F811
            return graphed(None if fin.values.data_ptr() == graphed.inp.data_ptr() else fin.values)
    batched = None
    if a.lanes:
        if a.streamed or sharded:
            raise SystemExit("--lanes runs the single-GPU in-memory round trip")
        batched = sc.BatchedRoundTrip(t, lanes=a.lanes, spin=a.spin, real=a.real)
        outb = torch.empty((a.lanes, *f.values.shape), dtype=f.values.dtype, device=dev)

        def step(fin):  # noqa: F811
            maps = fin.values if fin.values.dim() == 3 else [fin.values] * a.lanes
            batched(maps, out=outb)
            return sc.SphereSignal(f.grid, f.spin, outb[0], real=a.real)

    if sharded and a.streamed:
        from paper_1511_05578_b200.dist import roundtrip_sharded_streamed
        K_fin = 2 * Ljs[-1] - 1
        rows = max(1, int(a.slab_gb * (1 << 30)) // (K_fin * K_fin * 16))

        def step(fin):  # noqa: F811
            g = roundtrip_sharded_streamed(fin, t, slab_rows=rows)
            return g if g is not None else fin
    elif sharded:
        from paper_1511_05578_b200.dist import analyze_sharded, synthesize_sharded

        def step(fin):  # noqa: F811
            c = analyze_sharded(fin, t, real=a.real)
            g = synthesize_sharded(c, t)
            return g if g is not None else fin

    # first map: context, per-L tables (Delta wedge, quadrature table, DFT
    # tables), plans and the first round trip -- what a one-map user pays
    ctx.profile(True)
    g = step(f)
    torch.cuda.synchronize()
    first_map_ms = (time.perf_counter() - t_first0) * 1e3
    ctx.profile(False)
    first_prof = ctx.profile_report()
    table_ms = sum(v[1] for k, v in first_prof.items() if k.endswith("_build") or k.startswith("delta"))
    for _ in range(max(0, a.warmup - 1)):
        g = step(f)
    torch.cuda.synchronize()
    rt_err = float((g.values - f.values).abs().max() / f.values.abs().max())

    hbm_peak = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            hbm_peak = float(json.load(fh)["hbm_gbs"])
        hbm_src = "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        hbm_peak = 6650.0
        hbm_src = "B200_PROFILING.md fallback"
    dfma_peak = ctx.fp64_peak_tflops()
    dmma_peak = ctx.dmma_peak_tflops()
    fp64_peak = max(dfma_peak, dmma_peak)

    # ---------------- timed region (device-resident input) ----------------
    stream = torch.cuda.current_stream()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.profile_report()  # clear
    ctx.profile(True)
    l0 = ctx.launch_count()
    clk = ClockSampler(local)
    clk.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(a.steps):
        g = step(f)
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ctx.profile(False)
    launches = ctx.launch_count() - l0
    prof = ctx.profile_report()
    if batched is not None:
        launches = batched.kernels_per_map * a.lanes * a.steps
        ctx.profile(True)
        for _ in range(a.steps * a.lanes):
            eager_step(f)
        torch.cuda.synchronize()
        ctx.profile(False)
        prof = {k: (n, ms / a.lanes) for k, (n, ms) in ctx.profile_report().items()}
    elif graphed is not None:
        # replays make no library calls: count the captured kernels, and take the
        # stage profile from the same number of eager steps (profiled after timing)
        launches = graphed.kernels_per_replay * a.steps
        ctx.profile(True)
        for _ in range(a.steps):
            eager_step(f)
        torch.cuda.synchronize()
        ctx.profile(False)
        prof = ctx.profile_report()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        lt = torch.tensor([launches], device=dev, dtype=torch.float64)
        dist.all_reduce(lt, op=dist.ReduceOp.SUM)
        launches = int(lt.item())
    ms_per_step = ms / a.steps
    maps_per_step = 1 if sharded else world * max(1, a.lanes)
    value = maps_per_step * a.steps / (ms * 1e-3)

    # ---------------- e2e: host buffers through the public API ----------------
    e2e = None
    if not a.no_e2e:
        bshape = ((a.lanes,) if a.lanes else ()) + tuple(f.values.shape)
        host_in = torch.empty(bshape, dtype=f.values.dtype, pin_memory=True)
        host_in.copy_(f.values.cpu().expand(bshape))
        host_out = torch.empty_like(host_in, pin_memory=True)
        dev_in = torch.empty(bshape, dtype=f.values.dtype, device=dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            dev_in.copy_(host_in, non_blocking=True)
            if a.lanes:
                step(_Batch(dev_in))
                host_out.copy_(outb, non_blocking=True)
            else:
                fin = sc.SphereSignal(f.grid, f.spin, dev_in, real=a.real)
                gg = step(fin)
                host_out.copy_(gg.values, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        nb = host_in.numel() * host_in.element_size()
        e2e = {"value": maps_per_step * a.steps / (ems * 1e-3), "unit": "maps/s", "h2d_bytes_per_step": nb,
               "d2h_bytes_per_step": nb, "ms_per_step": ems / a.steps}

    roof = stage_roofline(a, prof, Ljs, hbm_peak, fp64_peak, dmma_peak)
    roof["peak_source"] = roof.get("peak_source", "") if roof.get("bound") != "hbm" else hbm_src
    t_roof = max(B_alg / (hbm_peak * 1e9 * world), F_alg / (fp64_peak * 1e12 * world))
    line = {
        "metric": "curvelet analysis+synthesis maps/s",
        "value": value,
        "unit": "maps/s",
        "n_gpus": world,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None,
        "dtype": "f64" if a.real else "c128",
        "data": "synthetic (seeded Gaussian f_lm, C_l=(l+1)^-2)",
        "config": arm_config(a, p, Ljs, world, sharded, maps_per_step),
        "roofline": roof,
        "paper_roofline": {"B_alg_GB": B_alg / 1e9, "F_alg_TF": F_alg / 1e12, "t_roof_ms": t_roof * 1e3,
                           "frac": t_roof * 1e3 * max(1, a.lanes) / ms_per_step, "fp64_peak_tflops": fp64_peak,
                           "fp64_peak_source": "max(in-run DFMA loop %.2f TF, in-run DMMA m8n8k4 loop %.2f TF) "
                                               "per GPU, x n_gpus" % (dfma_peak, dmma_peak),
                           "hbm_peak_gbs": hbm_peak, "hbm_peak_source": hbm_src},
        "stages_ms_per_step": {k: v[1] / a.steps for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])},
        "roundtrip_rel_err": rt_err,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
        "first_map_ms": first_map_ms,
        "first_map": {"ms": first_map_ms, "table_build_ms": table_ms,
                      "what": "context + per-L tables (Delta wedge, beta-quadrature table, DFT tables) + the first "
                              "round trip, host wall clock; excluded from the timed region like the reference's "
                              "cached Delta / kernel FFTs (cli.py:257-263)",
                      "stages_ms": {k: v[1] for k, v in sorted(first_prof.items(), key=lambda kv: -kv[1][1])[:6]}},
        "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9 + ctx.workspace_bytes() / 1e9,
    }
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        from oracle import cpu_sample

        def gpu_ms_at(L):
            pp = sc.TilingParams(L, a.spin, a.lam, a.jmin)
            tt_ = sc.build_tiling(pp)
            fl = sc.sht_inverse(sc.HarmonicCoeffs(L, a.spin, gaussian_flm(L, a.spin, a.seed, a.spin == 0)))
            for _ in range(2):
                sc.synthesize(sc.analyze(fl, tt_), tt_)
            torch.cuda.synchronize()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            q0.record()
            for _ in range(5):
                sc.synthesize(sc.analyze(fl, tt_), tt_)
            q1.record()
            torch.cuda.synchronize()
            return q0.elapsed_time(q1) / 5

        measured = None if a.no_measured_cpu or a.real else measured_cpu_roundtrip(a, gpu_ms_at)
        line["cpu_baseline"] = cpu_sample.calibrated_baseline(a.L, a.spin, a.lam, a.jmin, a.real, measured)
    if a.profile_json and rank == 0:
        with open(a.profile_json, "w") as fh:
            json.dump(line, fh, indent=1)
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_reference(a):
    """The reference's algorithm on the host CPU (oracle port, numpy +
    scipy.fft with every host thread), rank 0 only.  A full L=1024 reference
    round trip needs >147 GB of host RAM and ~40 min, so each STEP times a
    bounded sample of the same map -- one n-chunk / beta-block piece per
    distinct scale size plus both SHTs (oracle/cpu_sample.py) -- and scales it
    by the piece counts.  The first warm-up step also times one FULL round trip
    at L=256, which calibrates the sampler.  ms_per_step is the real wall time
    of a step (the sample); value = 1 / (calibrated seconds per map), i.e.
    the map fraction a step covers divided by its wall time."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import cpu_sample
    p, Ljs, _, _ = algorithmic_work(a)
    world = int(os.environ.get("WORLD_SIZE", a.gpus))
    sharded = world > 1 and not a.maps_per_rank
    measured = None
    if not a.real and not a.no_measured_cpu:
        measured = measured_cpu_roundtrip_host_only(a)
    raw, walls = [], []
    t_run0 = time.perf_counter()
    for i in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        cb = cpu_sample.baseline(a.L, a.spin, a.lam, a.jmin, a.real)
        if i >= a.warmup:
            raw.append(cb["seconds_per_map"])
            walls.append(time.perf_counter() - t0)
    est = statistics.median(raw)
    factor = 1.0
    cal = None
    if measured is not None:
        est_m = sorted(cpu_sample.baseline(measured["L"], a.spin, a.lam, a.jmin, a.real)["seconds_per_map"]
                       for _ in range(3))[1]
        factor = measured["all_cores"]["s_per_map"] / est_m
        cal = {"L": measured["L"], "measured_s_per_map": measured["all_cores"]["s_per_map"],
               "estimated_s_per_map": est_m, "factor": factor}
    sec = est * factor
    value = 1.0 / sec
    step_s = statistics.median(walls)
    cb = {"value": value, "unit": "maps/s", "seconds_per_map": sec, "cores": os.cpu_count() or 1, "kind": "port",
          "sample": cb["sample"] + (f"; calibrated x{factor:.3f} by a full round trip at L=256" if cal else ""),
          "estimate_uncalibrated_s_per_map": est, "estimate_spread_s_per_map": raw, "calibration": cal,
          "measured": measured, "per_scale_seconds": cb["per_scale_seconds"]}
    line = {
        "impl": "reference",
        "metric": "curvelet analysis+synthesis maps/s",
        "value": value,
        "unit": "maps/s",
        "n_gpus": a.gpus,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": step_s * 1e3,
        "map_fraction_per_step": step_s / sec,
        "run_wall_s": time.perf_counter() - t_run0,
        "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None,
        "dtype": "f64" if a.real else "c128",
        "data": "synthetic (seeded Gaussian f_lm, C_l=(l+1)^-2)",
        # the GPU arm's config, key for key (the driver compares the two lines)
        "config": arm_config(a, p, Ljs, world, sharded, 1 if sharded else world * max(1, a.lanes)),
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "maps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def measured_cpu_roundtrip_host_only(a):
    """measured_cpu_roundtrip without the GPU column (reference arm: all cores only)."""
    from scipy import fft as sfft
    from oracle import scurve_oracle as orc
    from paper_1511_05578_b200 import tiling as T
    L = 256
    p = T.TilingParams(L, a.spin, a.lam, a.jmin)
    t = T.build_tiling(p)
    psi = [T.curvelet_harmonics(t, j) for j in range(p.j_min, p.j_max + 1)]
    f = orc.sht_inverse(gaussian_flm(L, a.spin, a.seed, a.spin == 0), L, a.spin)
    workers = os.cpu_count() or 1
    with sfft.set_workers(workers):
        t0 = time.perf_counter()
        smap, scales = orc.analyze(f, L, a.spin, a.lam, a.jmin, p.j_max, psi, t.scaling)
        orc.synthesize(smap, scales, L, a.spin, a.lam, a.jmin, p.j_max, psi, t.scaling)
        sec = time.perf_counter() - t0
    return {"L": L, "all_cores": {"cores": workers, "s_per_map": sec}}


if __name__ == "__main__":
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
