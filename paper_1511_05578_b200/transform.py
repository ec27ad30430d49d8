"""Curvelet analysis and synthesis — the drop-in entry points.

Mirrors ``scurve.transform`` (transform.py:63-253): ``analyze``,
``synthesize``, ``analyze_real``, ``synthesize_real``, ``CurveletCoeffs``,
``scale_band_limit``, ``scaling_band_limit`` — same arguments, checks
(ValueError on band-limit / spin / frame / params mismatch) and output
layouts.  Every arithmetic step runs in libscurve_b200.so on the device;
the Python layer only sequences the calls, allocates outputs and validates.

Ordering is the reference's: scales coarse -> fine, then the scaling part,
so the synthesis accumulation is deterministic.
"""

from __future__ import annotations

import math
import threading
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _cabi
from .so3 import (CurveletWignerCoeffs, SO3Grid, WignerCoeffs, SO3Signal, so3_forward_curvelet,
                  so3_forward_curvelet_real, so3_forward_curvelet_slab, so3_inverse_curvelet,
                  so3_inverse_curvelet_real, so3_inverse_curvelet_slab)
from .sphere import (HarmonicCoeffs, SphereGrid, SphereSignal, sht_forward, sht_forward_real,
                     sht_inverse, sht_inverse_real)
from .tiling import Tiling, TilingParams, curvelet_harmonics

__all__ = [
    "CurveletCoeffs",
    "BatchedRoundTrip",
    "GraphedRoundTrip",
    "analyze",
    "analyze_real",
    "analyze_north_validation",
    "rotate_from_north",
    "rotate_to_north",
    "roundtrip_streamed",
    "scale_band_limit",
    "scaling_band_limit",
    "synthesize",
    "synthesize_real",
]


def scale_band_limit(params: TilingParams, j: int) -> int:
    """min(ceil(lam^(j+1)), L) (transform.py:63-67)."""
    if not params.j_min <= j <= params.j_max:
        raise ValueError(f"scale {j} outside [{params.j_min}, {params.j_max}]")
    return min(math.ceil(params.lam ** (j + 1)), params.band_limit)


def scaling_band_limit(params: TilingParams) -> int:
    """min(ceil(lam^j_min), L) (transform.py:70-72)."""
    return min(math.ceil(params.lam ** params.j_min), params.band_limit)


@dataclass
class CurveletCoeffs:
    """Scale signals plus the low-frequency residue (transform.py:75-101)."""

    params: TilingParams
    frame: str
    scaling: SphereSignal
    scales: list
    multires: bool = True
    real: bool = False

    def __post_init__(self):
        if self.frame not in ("unrotated", "north"):
            raise ValueError(f"unknown frame {self.frame!r}")
        if len(self.scales) != self.params.scale_count:
            raise ValueError(f"expected {self.params.scale_count} scale signals, got {len(self.scales)}")

    def scale(self, j: int):
        if not self.params.j_min <= j <= self.params.j_max:
            raise ValueError(f"scale {j} out of range")
        return self.scales[j - self.params.j_min]


# ---------------------------------------------------------------------------
# tiling arrays on the device (uploaded once per Tiling object)
# ---------------------------------------------------------------------------
_tcache: dict = {}
_tcache_lock = threading.Lock()


class _DevTiling:
    def __init__(self, t, device):
        p = t.params
        self.psi = {}
        for j in range(p.j_min, p.j_max + 1):
            pos, neg = curvelet_harmonics(t, j)
            # np.array copies: tiling arrays may be read-only views (frozen reference Tiling)
            self.psi[j] = (torch.as_tensor(np.array(pos, dtype=np.float64), device=device),
                           torch.as_tensor(np.array(neg, dtype=np.float64), device=device))
        self.scaling = torch.as_tensor(np.array(t.scaling, dtype=np.float64), device=device)


def device_tiling(t, device) -> _DevTiling:
    key = (id(t), str(device))
    with _tcache_lock:
        hit = _tcache.get(key)
        if hit is not None and hit[0]() is t:
            return hit[1]
        d = _DevTiling(t, device)
        try:
            ref = weakref.ref(t)
        except TypeError:
            ref = lambda t=t: t  # noqa: E731
        _tcache[key] = (ref, d)
        return d


def _check_signal(f: SphereSignal, t) -> None:
    p = t.params
    if f.grid.band_limit != p.band_limit:
        raise ValueError(f"signal band limit {f.grid.band_limit} does not match tiling {p.band_limit}")
    if f.spin != p.spin:
        raise ValueError(f"signal spin {f.spin} does not match tiling spin {p.spin}")


def _scale_wigner(ctx, flm: HarmonicCoeffs, dt: _DevTiling, j: int, Lj: int) -> CurveletWignerCoeffs:
    """transform.py:104-115 on the device."""
    pos, neg = dt.psi[j]
    w = torch.empty((2, Lj, 2 * Lj - 1), dtype=torch.complex128, device=flm.values.device)
    ctx.call("scale_product", flm.band_limit, Lj, _cabi.ptr(flm.values), _cabi.ptr(pos), _cabi.ptr(neg),
             _cabi.ptr(w))
    return CurveletWignerCoeffs(Lj, w)


def _scaling_coeffs(ctx, flm: HarmonicCoeffs, dt: _DevTiling, Ls: int, real: bool) -> HarmonicCoeffs:
    """transform.py:128-136 on the device."""
    out = torch.empty(Ls * Ls, dtype=torch.complex128, device=flm.values.device)
    ctx.call("scaling_product", flm.band_limit, Ls, _cabi.ptr(flm.values), _cabi.ptr(dt.scaling), _cabi.ptr(out))
    return HarmonicCoeffs(Ls, 0, out, real=real)


class _MapPlan:
    """Host-side argument arrays of scv_analyze / scv_synthesize for one (tiling, device,
    multires): band limits and device pointers of the kernel columns, built once."""

    def __init__(self, t, dt: _DevTiling, multires: bool):
        import ctypes
        p = t.params
        L = p.band_limit
        self.Ljs = [scale_band_limit(p, j) if multires else L for j in range(p.j_min, p.j_max + 1)]
        self.Ls = scaling_band_limit(p) if multires else L
        n = len(self.Ljs)
        self.n = n
        self.Lj_arr = (ctypes.c_int * n)(*self.Ljs)
        self.pos_arr = (ctypes.c_void_p * n)(*[dt.psi[j][0].data_ptr() for j in range(p.j_min, p.j_max + 1)])
        self.neg_arr = (ctypes.c_void_p * n)(*[dt.psi[j][1].data_ptr() for j in range(p.j_min, p.j_max + 1)])
        self.work_bytes = int(_cabi.load_library().scv_map_work_bytes(L, max(self.Ljs, default=1), self.Ls))
        self.sig_arr_t = ctypes.c_void_p * n


def _map_plan(t, dt: _DevTiling, multires: bool) -> _MapPlan:
    plans = dt.__dict__.setdefault("_map_plans", {})
    plan = plans.get(bool(multires))
    if plan is None:
        plan = plans[bool(multires)] = _MapPlan(t, dt, multires)
    return plan


def _analyze_stages(f: SphereSignal, t, multires: bool, real: bool, scale_out=None) -> CurveletCoeffs:
    """The scale loop driven from Python, one C call per stage (the path until r05; kept for a
    real-flagged signal analysed on the complex path and as the comparator of the whole-map call)."""
    _check_signal(f, t)
    p = t.params
    L = p.band_limit
    dev = f.values.device
    ctx = _cabi.context(dev)
    dt = device_tiling(t, dev)
    flm = sht_forward_real(f) if real else sht_forward(f)
    scales = []
    for j in range(p.j_min, p.j_max + 1):
        Lj = scale_band_limit(p, j) if multires else L
        w = _scale_wigner(ctx, flm, dt, j, Lj)
        buf = scale_out[j - p.j_min] if scale_out is not None else None
        inv = so3_inverse_curvelet_real if real else so3_inverse_curvelet
        scales.append(inv(w, SO3Grid(Lj, Lj, Lj), out=buf))
    Ls = scaling_band_limit(p) if multires else L
    s = _scaling_coeffs(ctx, flm, dt, Ls, real)
    scaling_sig = sht_inverse_real(s) if real else sht_inverse(s)
    return CurveletCoeffs(p, "unrotated", scaling_sig, scales, multires, real=real)


def _analyze(f: SphereSignal, t, multires: bool, real: bool, scale_out=None) -> CurveletCoeffs:
    """One scv_analyze call (the library walks the scales); bit-identical to _analyze_stages."""
    if f.real != real:
        return _analyze_stages(f, t, multires, real, scale_out)
    _check_signal(f, t)
    p = t.params
    L = p.band_limit
    if abs(p.spin) >= L:
        raise ValueError(f"spin {p.spin} out of range for band limit {L}")
    dev = f.values.device
    ctx = _cabi.context(dev)
    dt = device_tiling(t, dev)
    plan = _map_plan(t, dt, multires)
    dtype = torch.float64 if real else torch.complex128
    if scale_out is not None and len(scale_out) != plan.n:
        raise ValueError(f"expected {plan.n} scale_out buffers, got {len(scale_out)}")
    outs = []
    for i, Lj in enumerate(plan.Ljs):
        K = 2 * Lj - 1
        if scale_out is None or scale_out[i] is None:
            buf = torch.empty((K, Lj, K), dtype=dtype, device=dev)
        else:
            buf = _cabi.checked(scale_out[i], dtype, (K, Lj, K), dev, "out")
        outs.append(buf)
    Ls = plan.Ls
    smap = torch.empty((Ls, 2 * Ls - 1), dtype=dtype, device=dev)
    work = torch.empty(plan.work_bytes, dtype=torch.uint8, device=dev)
    sig_arr = plan.sig_arr_t(*[b.data_ptr() for b in outs])
    ctx.call("analyze", L, p.spin, 1 if real else 0, plan.n, plan.Lj_arr, plan.pos_arr, plan.neg_arr,
             _cabi.ptr(dt.scaling), Ls, _cabi.ptr(f.values), sig_arr, _cabi.ptr(smap), _cabi.ptr(work),
             plan.work_bytes)
    scales = [SO3Signal(SO3Grid(Lj, Lj, Lj), b, real=real) for Lj, b in zip(plan.Ljs, outs)]
    return CurveletCoeffs(p, "unrotated", SphereSignal(SphereGrid(Ls), 0, smap, real=real), scales, multires,
                          real=real)


def analyze(f: SphereSignal, t: Tiling, multires: bool = True, scale_out=None) -> CurveletCoeffs:
    """Decompose a band-limited spin signal into directional scale signals
    (transform.py:139-152).  ``scale_out`` optionally supplies preallocated
    (K_j, L_j, K_j) output tensors, one per scale (device-resident reuse)."""
    return _analyze(f, t, multires, False, scale_out)


def analyze_real(f: SphereSignal, t: Tiling, multires: bool = True, scale_out=None) -> CurveletCoeffs:
    """Half-spectrum analysis of a real signal (transform.py:190-210)."""
    if not f.real:
        raise ValueError("analyze_real requires a real-flagged signal")
    return _analyze(f, t, multires, True, scale_out)


def _check_coeffs(c: CurveletCoeffs, t) -> None:
    p = t.params
    if c.params != p:
        raise ValueError("coefficients were built for a different tiling")
    if c.frame != "unrotated":
        raise ValueError("synthesis needs unrotated coefficients; apply rotate_from_north first")
    L = p.band_limit
    for j in range(p.j_min, p.j_max + 1):
        sig = c.scale(j)
        expected = scale_band_limit(p, j) if c.multires else L
        if sig.grid.L != expected:
            raise ValueError(f"scale {j} stored at band limit {sig.grid.L}, expected {expected}")


def _synthesize_stages(c: CurveletCoeffs, t, real: bool) -> SphereSignal:
    """The scale loop driven from Python, one C call per stage (comparator of the whole-map call,
    and the path for coefficient sets whose flags or layouts the whole-map call does not take)."""
    _check_coeffs(c, t)
    p = t.params
    L = p.band_limit
    dev = c.scaling.values.device
    ctx = _cabi.context(dev)
    dt = device_tiling(t, dev)
    acc = torch.zeros(L * L, dtype=torch.complex128, device=dev)
    wbuf = None
    for j in range(p.j_min, p.j_max + 1):
        sig = c.scale(j)
        Lj = sig.grid.L
        need = 2 * Lj * (2 * Lj - 1)
        if wbuf is None or wbuf.numel() < need:
            wbuf = torch.empty(need, dtype=torch.complex128, device=dev)
        wv = wbuf[:need].view(2, Lj, 2 * Lj - 1)
        w = so3_forward_curvelet_real(sig, out=wv) if real else so3_forward_curvelet(sig, out=wv)
        pos, neg = dt.psi[j]
        ctx.call("accumulate", L, Lj, _cabi.ptr(w.values), _cabi.ptr(pos), _cabi.ptr(neg), _cabi.ptr(acc))
    slm = sht_forward_real(c.scaling) if real else sht_forward(c.scaling)
    ctx.call("accumulate_scaling", L, slm.band_limit, _cabi.ptr(slm.values), _cabi.ptr(dt.scaling), _cabi.ptr(acc))
    ctx.call("finish_acc", L, p.spin, 1 if real else 0, _cabi.ptr(acc))
    if real:
        return sht_inverse_real(HarmonicCoeffs(L, 0, acc, real=True, trusted=True))
    return sht_inverse(HarmonicCoeffs(L, p.spin, acc, trusted=True))


def _synthesize(c: CurveletCoeffs, t, real: bool) -> SphereSignal:
    """One scv_synthesize call (the library walks the scales); bit-identical to _synthesize_stages."""
    _check_coeffs(c, t)
    p = t.params
    L = p.band_limit
    dev = c.scaling.values.device
    dtype = torch.float64 if real else torch.complex128
    sigs = [c.scale(j) for j in range(p.j_min, p.j_max + 1)]
    dt = device_tiling(t, dev)
    plan = _map_plan(t, dt, c.multires)
    plain = (c.scaling.real == real and c.scaling.spin == 0 and c.scaling.grid.band_limit == plan.Ls
             and c.scaling.values.dtype == dtype
             and all(s.real == real and s.values.dtype == dtype and s.values.device == dev and
                     (s.grid.L, s.grid.M, s.grid.N) == (Lj, Lj, Lj) for s, Lj in zip(sigs, plan.Ljs)))
    if not plain:
        return _synthesize_stages(c, t, real)
    ctx = _cabi.context(dev)
    for s, Lj in zip(sigs, plan.Ljs):
        _cabi.checked(s.values, dtype, (2 * Lj - 1, Lj, 2 * Lj - 1), dev, "signal values")
    Ls = plan.Ls
    _cabi.checked(c.scaling.values, dtype, (Ls, 2 * Ls - 1), dev, "scaling values")
    out = torch.empty((L, 2 * L - 1), dtype=dtype, device=dev)
    work = torch.empty(plan.work_bytes, dtype=torch.uint8, device=dev)
    sig_arr = plan.sig_arr_t(*[s.values.data_ptr() for s in sigs])
    ctx.call("synthesize", L, p.spin, 1 if real else 0, plan.n, plan.Lj_arr, plan.pos_arr, plan.neg_arr,
             _cabi.ptr(dt.scaling), Ls, sig_arr, _cabi.ptr(c.scaling.values), _cabi.ptr(out), _cabi.ptr(work),
             plan.work_bytes)
    return SphereSignal(SphereGrid(L), 0 if real else p.spin, out, real=real)


def synthesize(c: CurveletCoeffs, t: Tiling) -> SphereSignal:
    """Reassemble the sphere signal from its scale signals (transform.py:155-187)."""
    return _synthesize(c, t, False)


def synthesize_real(c: CurveletCoeffs, t: Tiling) -> SphereSignal:
    """Synthesis matching analyze_real (transform.py:213-253)."""
    if not c.real:
        raise ValueError("synthesize_real requires real-flagged coefficients")
    return _synthesize(c, t, True)


# ---------------------------------------------------------------------------
# beta-slab streamed round trip
# ---------------------------------------------------------------------------
def _slab_streamable(Lj: int) -> bool:
    """Scales the beta-slab kernels take (include/scurve_b200.h): complex
    path, prime-factor K = 2^k - 1, 128 <= L_j <= 2048."""
    K = 2 * Lj - 1
    return 128 <= Lj <= 2048 and (K & (K + 1)) == 0


def _syn_chunk_rows(Lj: int) -> int:
    """Beta rows per synthesis launch pair inside the library
    (scv_syn_chunk_rows, so3.cu)."""
    return max(1, int(_cabi.load_library().scv_syn_chunk_rows(int(Lj))))


def roundtrip_streamed(f: SphereSignal, t: Tiling, multires: bool = True, slab_bytes: int = 8 << 30,
                       consumer=None):
    """``synthesize(analyze(f, t), t)`` without holding the coefficients.

    The reference's round trip (``cli.cmd_roundtrip``, cli.py:227-246) keeps
    every scale signal in memory: 147 GB at L=1024 and 1.18 TB at L=2048
    (BASELINE config C5), more than one B200 holds.  Here each large scale
    (prime-factor K, 128 <= L_j <= 2048) is analysed in beta slabs of at most
    ``slab_bytes``; every slab is handed to ``consumer(j, slab)`` (an
    ``SO3Slab``: the rows [b0, b0+nb) of scale j's signal, valid only during
    the call) and then folded into scale j's Wigner coefficients by the slab
    synthesis, before the next slab overwrites the buffer.  Smaller scales
    run whole (``consumer(j, SO3Signal)``).  The scaling signal is passed as
    ``consumer("scaling", SphereSignal)``.

    Slab heights are multiples of the library's synthesis chunk, so the
    summation order is the whole-scale one and the result is bit-identical
    to ``synthesize(analyze(f, t), t)``.  Returns the reconstructed signal.
    """
    _check_signal(f, t)
    p = t.params
    L = p.band_limit
    dev = f.values.device
    ctx = _cabi.context(dev)
    dt = device_tiling(t, dev)
    flm = sht_forward(f)
    acc = torch.zeros(L * L, dtype=torch.complex128, device=dev)
    slab_buf = None
    for j in range(p.j_min, p.j_max + 1):
        Lj = scale_band_limit(p, j) if multires else L
        K = 2 * Lj - 1
        grid = SO3Grid(Lj, Lj, Lj)
        w = _scale_wigner(ctx, flm, dt, j, Lj)
        if _slab_streamable(Lj):
            ch = _syn_chunk_rows(Lj)
            nb = max(ch, (slab_bytes // (K * K * 16)) // ch * ch)
            nb = min(nb, Lj)
            need = K * nb * K
            if slab_buf is None or slab_buf.numel() < need:
                slab_buf = None
                slab_buf = torch.empty(need, dtype=torch.complex128, device=dev)
            W = None
            for b0 in range(0, Lj, nb):
                nbb = min(nb, Lj - b0)
                out = slab_buf[: K * nbb * K].view(K, nbb, K)
                slab = so3_inverse_curvelet_slab(w, grid, b0, nbb, out=out)
                if consumer is not None:
                    consumer(j, slab)
                if W is None:
                    W = so3_forward_curvelet_slab(slab)
                else:
                    so3_forward_curvelet_slab(slab, out=W.values, accumulate=True)
        else:
            sig = so3_inverse_curvelet(w, grid)
            if consumer is not None:
                consumer(j, sig)
            W = so3_forward_curvelet(sig)
            del sig
        pos, neg = dt.psi[j]
        ctx.call("accumulate", L, Lj, _cabi.ptr(W.values), _cabi.ptr(pos), _cabi.ptr(neg), _cabi.ptr(acc))
    Ls = scaling_band_limit(p) if multires else L
    scaling_sig = sht_inverse(_scaling_coeffs(ctx, flm, dt, Ls, False))
    if consumer is not None:
        consumer("scaling", scaling_sig)
    slm = sht_forward(scaling_sig)
    ctx.call("accumulate_scaling", L, slm.band_limit, _cabi.ptr(slm.values), _cabi.ptr(dt.scaling), _cabi.ptr(acc))
    ctx.call("finish_acc", L, p.spin, 0, _cabi.ptr(acc))
    return sht_inverse(HarmonicCoeffs(L, p.spin, acc, trusted=True))


# ---------------------------------------------------------------------------
# frame rotation (transform.py:256-297), csrc/rotate.cu
# ---------------------------------------------------------------------------
def _rotation_angle(j: int, t: Tiling) -> float:
    p = t.params
    if not p.j_min <= j <= p.j_max:
        raise ValueError(f"scale {j} outside [{p.j_min}, {p.j_max}]")
    return float(t.angles[j - p.j_min])


def rotate_to_north(w: CurveletWignerCoeffs, j: int, t: Tiling) -> WignerCoeffs:
    """Move a scale's coefficients to the frame of the pole-centred function
    (transform.py:256-277): dense planes outer(w[+l], d_{.,+l}(theta_j)) +
    outer(w[-l], d_{.,-l}(theta_j)), one warp per plane row (k_rot_to_north)."""
    if not isinstance(w, CurveletWignerCoeffs):
        raise TypeError("rotate_to_north expects sparse coefficients")
    theta = _rotation_angle(j, t)
    L = w.band_limit
    ctx = _cabi.context(w.values.device)
    out = WignerCoeffs(L, values=torch.empty(L * (4 * L * L - 1) // 3, dtype=torch.complex128,
                                             device=w.values.device))
    ctx.call("rotate_to_north", L, theta, _cabi.ptr(w.values), _cabi.ptr(out.values))
    return out


def rotate_from_north(w: WignerCoeffs, j: int, t: Tiling) -> CurveletWignerCoeffs:
    """Inverse of rotate_to_north, exact on its image (transform.py:280-297):
    w[+l] = plane_l d_{.,+l}(theta_j), w[-l] = plane_l d_{.,-l}(theta_j)."""
    if not isinstance(w, WignerCoeffs):
        raise TypeError("rotate_from_north expects dense coefficients")
    theta = _rotation_angle(j, t)
    L = w.band_limit
    ctx = _cabi.context(w.values.device)
    out = torch.empty((2, L, 2 * L - 1), dtype=torch.complex128, device=w.values.device)
    ctx.call("rotate_from_north", L, theta, _cabi.ptr(w.values), _cabi.ptr(out))
    return CurveletWignerCoeffs(L, out)


# ---------------------------------------------------------------------------
# CUDA-graph replay of a fixed-shape round trip (launch-bound band limits)
# ---------------------------------------------------------------------------
class GraphedRoundTrip:
    """``analyze`` + ``synthesize`` of same-shape maps replayed from one CUDA graph.

    At small band limits (C1 L=64, C2 L=128) a round trip is ~100-200 short
    kernels and the host launch path dominates.  This captures the whole
    pipeline once.  Two eager passes on a side stream first build every
    per-L table, cuFFT plan and scratch buffer, so nothing allocates or
    synchronises during capture.  ``__call__`` then copies a map into the
    captured input and replays.  The outputs (``coeffs``, ``out``) are
    graph-owned tensors, overwritten by the next call.  Results are
    bit-identical to the eager calls (the same kernels on the same buffers;
    tests/test_graph.py).

    The graph holds raw pointers into its context's workspace (scratch
    slots, cuFFT work area, Delta and log-binomial tables), which the
    library grows and frees on demand.  By default the instance therefore
    owns a private context, so eager calls elsewhere can never move memory
    the graph replays against.  With ``private_context=False`` the shared
    per-device context is PINNED while the instance lives (``close()`` or
    garbage collection releases it): any call that would grow, free or trim
    a workspace buffer of that context raises ValueError instead.
    """

    def __init__(self, t: Tiling, spin: int = 0, real: bool = False, multires: bool = True,
                 private_context: bool = True):
        L = t.params.band_limit
        dev = torch.device("cuda", torch.cuda.current_device())
        dtype = torch.float64 if real else torch.complex128
        self.t, self.real = t, real
        self._pinned = False
        # a private context owns its scratch, so several instances can replay
        # concurrently on different streams (BatchedRoundTrip)
        self.ctx = _cabi.new_context(dev.index) if private_context else _cabi.context(dev)
        self.stream = torch.cuda.Stream(dev)
        self.inp = torch.zeros((L, 2 * L - 1), dtype=dtype, device=dev)
        f = SphereSignal(SphereGrid(L), spin, self.inp, real=real)
        if f.values.data_ptr() != self.inp.data_ptr():
            raise RuntimeError("captured input was copied")
        ana, syn = (analyze_real, synthesize_real) if real else (analyze, synthesize)
        with _cabi.using(self.ctx):
            self.stream.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(self.stream):
                for _ in range(2):
                    syn(ana(f, t, multires), t)
            torch.cuda.synchronize(dev)
            n0 = self.ctx.launch_count()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=self.stream):
                self.coeffs = ana(f, t, multires)
                self.out = syn(self.coeffs, t)
            self.kernels_per_replay = self.ctx.launch_count() - n0
        if not private_context:
            self.ctx.set_option("pin", 1)
            self._pinned = True

    def close(self) -> None:
        """Release the graph (and the pin on a shared context)."""
        if getattr(self, "_pinned", False):
            self._pinned = False
            self.ctx.set_option("pin", 0)
        self.graph = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launch(self, values=None) -> SphereSignal:
        """Replay on this instance's own stream, ordered after the caller's
        current stream; the caller joins with ``join()``."""
        cur = torch.cuda.current_stream(self.inp.device)
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            if values is not None:
                self.inp.copy_(values if isinstance(values, torch.Tensor) else torch.as_tensor(values),
                               non_blocking=True)
            self.graph.replay()
        return self.out

    def join(self) -> None:
        torch.cuda.current_stream(self.inp.device).wait_stream(self.stream)

    def __call__(self, values=None) -> SphereSignal:
        out = self.launch(values)
        self.join()
        return out


class BatchedRoundTrip:
    """Round trips of a batch of same-shape maps, ``lanes`` at a time in flight.

    Each lane is a GraphedRoundTrip with a private context and its own
    stream, so the lanes' kernels overlap on the GPU.  At small band limits a
    single map occupies a fraction of the 148 SMs, and concurrent lanes fill
    the rest (batched multi-map pipelining).  Map i of a
    batch goes to lane i mod lanes; results are copied out of the lane's
    graph-owned output before the lane is reused.
    """

    def __init__(self, t: Tiling, lanes: int = 4, spin: int = 0, real: bool = False, multires: bool = True):
        if lanes < 1:
            raise ValueError("lanes must be positive")
        self.lanes = [GraphedRoundTrip(t, spin, real, multires, private_context=True) for _ in range(lanes)]
        self.kernels_per_map = self.lanes[0].kernels_per_replay

    def __call__(self, maps, out: torch.Tensor | None = None) -> torch.Tensor:
        """maps: (B, L, 2L-1) tensor (device or host).  Returns (B, L, 2L-1) reconstructions."""
        n = len(maps)
        first = self.lanes[0].out.values
        if out is None:
            out = torch.empty((n, *first.shape), dtype=first.dtype, device=first.device)
        for i in range(n):
            lane = self.lanes[i % len(self.lanes)]
            g = lane.launch(maps[i])
            with torch.cuda.stream(lane.stream):
                out[i].copy_(g.values, non_blocking=True)
        for lane in self.lanes:
            lane.join()
        return out


def analyze_north_validation(f: SphereSignal, t: Tiling, j: int, max_band_limit: int = 32) -> SO3Signal:
    """Scale-j signal computed the slow way, through the dense frame
    (transform.py:300-322): scale coefficients, rotate_to_north, then the
    dense O(L^4) synthesis.  A cross-check of the fast path, hence the cap."""
    from .so3 import so3_inverse_general
    _check_signal(f, t)
    p = t.params
    if not p.j_min <= j <= p.j_max:
        raise ValueError(f"scale {j} outside [{p.j_min}, {p.j_max}]")
    Lj = scale_band_limit(p, j)
    if Lj > max_band_limit:
        raise ValueError(f"band limit {Lj} exceeds the dense validation cap {max_band_limit}")
    dev = f.values.device
    ctx = _cabi.context(dev)
    flm = sht_forward(f)
    w = _scale_wigner(ctx, flm, device_tiling(t, dev), j, Lj)
    dense = rotate_to_north(w, j, t)
    return so3_inverse_general(dense, SO3Grid(Lj, Lj, Lj))
