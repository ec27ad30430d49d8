"""Bounded-sample CPU timing of the reference algorithm — TEST/BENCH
INFRASTRUCTURE ONLY (imported by bench.py's cpu_baseline and --impl
reference legs, never by the product).

A full reference round trip at L=1024 needs >147 GB of host RAM and ~40 min
on 8 threads, so the baseline is measured on a
bounded sample of the SAME workload and scaled to one map: the reference
processes every scale in independent pieces — n-chunks of 16 planes
(so3.py:42, 272-283, 231-243) and beta-blocks of 8 for the gamma FFTs
(so3.py:185-192) — and the per-map time is the sum over pieces.  For each
scale we time one n-chunk (16 frequencies spread over the whole n range, so
plane sizes average out) and one beta-block of each FFT pass with the
oracle's own code at the real sizes, multiply by the piece counts, and add
the two SHTs (phi/theta FFT + weights convolution timed in full, the
per-degree Delta contraction timed on a spread sample of degrees).  The
Delta planes are random stand-ins of the right shape: the arithmetic cost
does not depend on their values.  scipy.fft runs with all host cores
(SCURVE_THREADS analogue); the Python loops are single-threaded, as in the
reference.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np
from scipy import fft as sfft

from . import scurve_oracle as orc


def _timed(fn):
    """min of two runs for short pieces (first-call overhead), one run otherwise"""
    t0 = time.perf_counter()
    fn()
    best = time.perf_counter() - t0
    if best < 0.5:
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


def _planes(L, ells, rng):
    P = {}
    for l in ells:
        if l not in P:
            P[l] = rng.standard_normal((2 * l + 1, 2 * l + 1))
    return P


def _spread_ns(L, k=16):
    ns = np.unique(np.round(np.linspace(-(L - 1), L - 1, k)).astype(int))
    return [int(n) for n in ns]


def _scale_seconds(Lj, real, rng, workers):
    K = 2 * Lj - 1
    ns = _spread_ns(Lj) if not real else sorted(set(abs(n) for n in _spread_ns(Lj)))
    planes = _planes(Lj, [abs(n) for n in ns], rng)
    w = (rng.standard_normal((2, Lj, K)) + 1j * rng.standard_normal((2, Lj, K)))
    nchunks = math.ceil((Lj if real else K) / 16)
    blk = min(8, Lj)
    with sfft.set_workers(workers):
        # analysis: one n-chunk of bin planes + ifft2 (so3.py:272-283)
        t_an = _timed(lambda: orc.so3_inverse_curvelet(w, planes, n_subset=ns)) * (16 / len(ns))
        slab = rng.standard_normal((K, blk, K)) + 1j * rng.standard_normal((K, blk, K))
        t_g = _timed(lambda: sfft.ifft(slab, axis=0))  # gamma IFFT block (so3.py:185-192)
        # synthesis: alpha + gamma FFT of a beta-block (so3.py:195-200)
        t_ag = _timed(lambda: sfft.fft(sfft.fft(slab, axis=2), axis=0))
        # synthesis: one n-chunk of the beta stage + contraction (so3.py:231-243)
        W1 = rng.standard_normal((len(ns), Lj, K)) + 1j * rng.standard_normal((len(ns), Lj, K))
        t_b = _timed(lambda: orc.so3_forward_rows(W1, ns, planes, Lj)) * (16 / len(ns))
    scale_blocks = Lj / blk
    if real:  # half the gamma spectrum
        t_g, t_ag = 0.5 * t_g, 0.5 * t_ag
    return nchunks * (t_an + t_b) + scale_blocks * (t_g + t_ag)


def _sht_seconds(L, rng, workers, spin=0):
    K = 2 * L - 1
    f = rng.standard_normal((L, K)) + 1j * rng.standard_normal((L, K))
    m = np.arange(-(L - 1), L)
    with sfft.set_workers(workers):
        def fft_part():
            G = np.fft.fftshift(sfft.fft(f, axis=1) / K, axes=1)
            orc.beta_to_bins(G, L, orc.sgn(m + spin), 0, 2 * math.pi)
        t_fft = _timed(fft_part)
        # per-degree contraction, sampled over a spread of degrees (sphere.py:174-181)
        ells = sorted(set(np.round(np.linspace(0, L - 1, min(L, 24))).astype(int).tolist()))
        Gw = rng.standard_normal((K, K)) + 1j * rng.standard_normal((K, K))
        c = L - 1

        def contract():
            for l in ells:
                D = np.ones((2 * l + 1, 2 * l + 1))
                u = D[:, l]
                blk = Gw[c - l:c + l + 1, c - l:c + l + 1]
                (D * u[:, None] * blk).sum(axis=0)
        t_c = _timed(contract)
        # sum over all degrees ~ mean sampled cost * L (cost grows as l^2: use the sample mean)
        t_c = t_c / len(ells) * L
        # inverse: bin-plane accumulation (same O(L^3) shape) + ifft2
        B = np.zeros((K, K), complex)
        t_i = _timed(lambda: sfft.ifft2(B)) + t_c
    return t_fft + t_c + t_i


def baseline(L, spin, lam, j_min, real, budget_s=20.0, seed=0):
    """Estimated seconds per map of the reference algorithm (oracle port) on
    this host, from the bounded per-piece sample described above."""
    from paper_1511_05578_b200.tiling import TilingParams
    workers = os.cpu_count() or 1
    p = TilingParams(L, spin, lam, j_min)
    rng = np.random.default_rng(seed)
    Ljs = [orc.scale_band_limit(L, lam, j) for j in range(p.j_min, p.j_max + 1)]
    t0 = time.perf_counter()
    per_scale = {}
    total = 0.0
    for Lj in sorted(set(Ljs)):
        s = _scale_seconds(Lj, real, rng, workers)
        per_scale[Lj] = s
        total += s * Ljs.count(Lj)
    Ls = orc.scaling_band_limit(L, lam, j_min)
    total += _sht_seconds(L, rng, workers, spin) + 2 * _sht_seconds(Ls, rng, workers)
    wall = time.perf_counter() - t0
    return {
        "value": 1.0 / total,
        "unit": "maps/s",
        "seconds_per_map": total,
        "cores": workers,
        "kind": "port",
        "sample": (f"one 16-frequency n-chunk (analysis planes+ifft2, synthesis beta stage+contraction) "
                   f"and one 8-row beta-block of the alpha/gamma FFTs per distinct scale band limit "
                   f"{sorted(set(Ljs))}, plus both SHTs at L={L} (contraction sampled over degrees); "
                   f"scaled by piece counts to one map; {wall:.1f} s of CPU sampling"),
        "per_scale_seconds": {str(k): v for k, v in per_scale.items()},
        "sampling_wall_s": wall,
    }


def calibrated_baseline(L, spin, lam, j_min, real, measured=None, repeats=2):
    """The bounded-sample estimate at L (median of `repeats` samples), and --
    when `measured` holds a full oracle round trip timed at L=256 on this host
    (bench.measured_cpu_roundtrip) -- the same estimator run at L=256, whose
    ratio to the measurement calibrates the L estimate (the sampler's piece
    timings miss per-call overheads and memory effects the full run has).
    `value` is the calibrated maps/s when a measurement exists, the raw
    estimate otherwise."""
    runs = [baseline(L, spin, lam, j_min, real) for _ in range(max(1, repeats))]
    runs.sort(key=lambda r: r["seconds_per_map"])
    mid = runs[len(runs) // 2]
    raw = mid["seconds_per_map"]
    out = dict(mid)
    out["estimate_uncalibrated_s_per_map"] = raw
    out["estimate_spread_s_per_map"] = [r["seconds_per_map"] for r in runs]
    out["sampling_wall_s"] = sum(r["sampling_wall_s"] for r in runs)
    if measured is not None:
        Lm = measured["L"]
        est_m = sorted(baseline(Lm, spin, lam, j_min, real)["seconds_per_map"] for _ in range(3))[1]
        meas = measured["all_cores"]["s_per_map"]
        factor = meas / est_m
        out["calibration"] = {"L": Lm, "measured_s_per_map": meas, "estimated_s_per_map": est_m,
                              "factor": factor,
                              "how": "seconds_per_map = raw estimate at L x (measured / estimated at L=%d)" % Lm}
        out["seconds_per_map"] = raw * factor
        out["value"] = 1.0 / (raw * factor)
        out["measured"] = measured
        out["sample"] = ("calibrated estimate: " + out["sample"] +
                         f"; x{factor:.3f} from a full round trip measured at L={Lm} on this host")
    return out
