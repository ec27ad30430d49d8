"""Sparsity report of curvelet coefficients on the device.

Mirror of the reference's ``scurve sparsity`` command (cli.py:268-320) and
``gini_coefficient`` (cli.py:59-70).  Per scale it gives the magnitude
histogram of |c| / max|c| over ``bins`` equal bins of [0, 1] (numpy's
``np.histogram`` rule, exact integer counts), the maximum magnitude, and the
Gini coefficient sum_i (2i - n - 1) x_(i) / (n sum x) of the sorted
magnitudes.  Everything runs in HBM (csrc/sparsity.cu): one magnitude pass,
one histogram pass, a device radix sort of the float64 magnitudes and one
deterministic reduction.

``sparsity_report(coeffs, bins)`` works on resident coefficients.
``sparsity_report_streamed(f, t, bins)`` analyses the map scale by scale in
beta slabs (as ``roundtrip_streamed`` does) and never holds the coefficient
volume.  At C4 (L=1024) it needs the two magnitude buffers of one finest scale
(2 x 34.3 GB) plus one slab, instead of the 147 GB of coefficients.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _cabi
from .so3 import SO3Grid, so3_inverse_curvelet, so3_inverse_curvelet_slab
from .sphere import SphereSignal, sht_forward
from .transform import (CurveletCoeffs, _check_signal, _scale_wigner, _slab_streamable, _syn_chunk_rows,
                        analyze, analyze_real, device_tiling, scale_band_limit)

__all__ = ["ScaleStats", "gini_coefficient", "scale_statistics", "sparsity_report", "sparsity_report_streamed"]


class ScaleStats:
    """Statistics of one scale's coefficient magnitudes."""

    def __init__(self, count: int, max_abs: float, counts: np.ndarray, gini):
        self.count, self.max_abs, self.counts, self.gini = count, max_abs, counts, gini


class _Accumulator:
    """Magnitudes of one scale gathered piece by piece into a device buffer."""

    def __init__(self, n: int, device):
        self.n = n
        self.mags = torch.empty(n, dtype=torch.float64, device=device)
        self.top = torch.zeros(1, dtype=torch.float64, device=device)
        self.off = 0
        self.ctx = _cabi.context(device)

    def add(self, values: torch.Tensor) -> None:
        v = values.contiguous().reshape(-1)
        k = v.numel()
        if self.off + k > self.n:
            raise ValueError("more magnitudes than the scale holds")
        dst = self.mags[self.off: self.off + k]
        self.ctx.call("abs_max", k, 1 if v.is_complex() else 0, _cabi.ptr(v), _cabi.ptr(dst), _cabi.ptr(self.top))
        self.off += k

    def finish(self, bins: int) -> ScaleStats:
        if self.off != self.n:
            raise ValueError(f"scale has {self.n} coefficients, {self.off} were added")
        return _stats(self.ctx, self.mags, self.top, bins)


def _stats(ctx, mags: torch.Tensor, top: torch.Tensor, bins: int) -> ScaleStats:
    n = mags.numel()
    dev = mags.device
    top_v = float(top.item())
    if top_v == 0.0:
        return ScaleStats(n, 0.0, None, None)
    edges = torch.from_numpy(np.linspace(0.0, 1.0, bins + 1)).to(dev)
    counts = torch.zeros(bins, dtype=torch.int64, device=dev)
    ctx.call("histogram", n, _cabi.ptr(mags), _cabi.ptr(top), bins, _cabi.ptr(edges), _cabi.ptr(counts))
    counts_h = counts.cpu().numpy()
    gini = _gini_inplace(ctx, mags)
    return ScaleStats(n, top_v, counts_h, gini)


def _gini_inplace(ctx, mags: torch.Tensor) -> float:
    """Sorts `mags` (destroyed) and returns the Gini coefficient."""
    import ctypes
    n = mags.numel()
    alt = torch.empty_like(mags)
    which = ctypes.c_int(0)
    ctx.call("sort_f64", n, _cabi.ptr(mags), _cabi.ptr(alt), ctypes.byref(which))
    srt = alt if which.value else mags
    out = torch.empty(2, dtype=torch.float64, device=mags.device)
    ctx.call("gini_sums", n, _cabi.ptr(srt), _cabi.ptr(out))
    num, total = (float(x) for x in out.cpu().numpy())
    del alt
    if n == 0 or total == 0.0:
        raise ValueError("Gini coefficient needs a non-empty, non-zero sample")
    return num / (n * total)


def gini_coefficient(magnitudes) -> float:
    """Concentration index of a non-negative sample: 0 flat, -> 1 peaked (cli.py:59-70)."""
    t = magnitudes if isinstance(magnitudes, torch.Tensor) else torch.as_tensor(np.asarray(magnitudes, dtype=float))
    t = t.to(device=torch.device("cuda", torch.cuda.current_device()), dtype=torch.float64).reshape(-1).clone()
    if t.numel() == 0:
        raise ValueError("Gini coefficient needs a non-empty, non-zero sample")
    if bool((t < 0).any()):
        raise ValueError("Gini coefficient needs non-negative values")
    return _gini_inplace(_cabi.context(t.device), t)


def scale_statistics(values: torch.Tensor, bins: int = 10) -> ScaleStats:
    """Histogram, max and Gini of |values| (one scale signal, device tensor)."""
    if bins < 1:
        raise ValueError("--bins must be at least 1")
    acc = _Accumulator(values.numel(), values.device)
    acc.add(values)
    return acc.finish(bins)


def _summary(params, bins, stats) -> tuple:
    """The reference's JSON summary and CSV rows (cli.py:278-313)."""
    edges = np.linspace(0.0, 1.0, bins + 1)
    rows, notes = [], []
    for j, st in stats:
        note = {"scale": j, "coefficients": int(st.count), "max_abs": st.max_abs}
        if st.max_abs == 0.0:
            note["gini"] = None
        else:
            note["gini"] = st.gini
            for b in range(bins):
                rows.append([params.band_limit, j, b, float(edges[b]), float(edges[b + 1]),
                             st.counts[b] / st.count])
        notes.append(note)
    summary = {"L": params.band_limit, "spin": params.spin, "lambda": params.lam, "j_min": params.j_min,
               "j_max": params.j_max, "bins": bins, "scales": notes}
    return summary, rows


def sparsity_report(coeffs: CurveletCoeffs, bins: int = 10) -> tuple:
    """(summary dict, csv rows) of `scurve sparsity` for resident coefficients."""
    if bins < 1:
        raise ValueError("--bins must be at least 1")
    p = coeffs.params
    stats = [(j, scale_statistics(coeffs.scale(j).values, bins)) for j in range(p.j_min, p.j_max + 1)]
    return _summary(p, bins, stats)


def sparsity_report_streamed(f: SphereSignal, t, bins: int = 10, slab_bytes: int = 8 << 30) -> tuple:
    """(summary, csv rows) of `scurve sparsity` for the analysis of `f`, streamed.

    Each scale's signal is produced in beta slabs (``so3_inverse_curvelet_slab``,
    the rows of ``analyze(f, t).scale(j)``), and every slab's magnitudes are
    appended to the scale's buffer.  The coefficient volume is never held.
    Small scales and real maps go through the whole-scale path.  A real map
    is analysed by the real path when it fits, as the reference's command
    does (``analyze_real`` if f.real).
    """
    if bins < 1:
        raise ValueError("--bins must be at least 1")
    _check_signal(f, t)
    p = t.params
    if f.real:
        c = analyze_real(f, t)
        return sparsity_report(c, bins)
    dev = f.values.device
    ctx = _cabi.context(dev)
    dt = device_tiling(t, dev)
    flm = sht_forward(f)
    stats = []
    slab_buf = None
    for j in range(p.j_min, p.j_max + 1):
        Lj = scale_band_limit(p, j)
        K = 2 * Lj - 1
        grid = SO3Grid(Lj, Lj, Lj)
        w = _scale_wigner(ctx, flm, dt, j, Lj)
        acc = _Accumulator(K * Lj * K, dev)
        if _slab_streamable(Lj):
            ch = _syn_chunk_rows(Lj)
            nb = min(Lj, max(ch, (slab_bytes // (K * K * 16)) // ch * ch))
            need = K * nb * K
            if slab_buf is None or slab_buf.numel() < need:
                slab_buf = None
                slab_buf = torch.empty(need, dtype=torch.complex128, device=dev)
            for b0 in range(0, Lj, nb):
                nbb = min(nb, Lj - b0)
                out = slab_buf[: K * nbb * K].view(K, nbb, K)
                acc.add(so3_inverse_curvelet_slab(w, grid, b0, nbb, out=out).values)
        else:
            acc.add(so3_inverse_curvelet(w, grid).values)
        stats.append((j, acc.finish(bins)))
        del acc
    return _summary(p, bins, stats)
