"""Sphere containers and the spin SHT on the MW grid (device tensors).

Drop-in mirror of ``scurve.sphere`` (sphere.py:36-260): same class and
function names, field names, shapes and ValueError conditions.  ``values``
are torch tensors on the CUDA device (numpy input is copied over); call
``.cpu().numpy()`` on them for host access.  The transforms run in
libscurve_b200.so (csrc/sht.cu, csrc/beta.cu).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from functools import cached_property

import numpy as np
import torch

from . import _cabi

__all__ = [
    "HarmonicCoeffs",
    "SphereGrid",
    "SphereSignal",
    "as_device",
    "lm_index",
    "sht_forward",
    "sht_forward_real",
    "sht_inverse",
    "sht_inverse_real",
]


def lm_index(ell: int, m: int) -> int:
    """ell^2 + ell + m (sphere.py:36-38)."""
    return ell * ell + ell + m


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1511_05578_b200 needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def as_device(x, dtype: torch.dtype) -> torch.Tensor:
    """numpy / torch -> contiguous device tensor of dtype (no copy if already so)."""
    if isinstance(x, torch.Tensor):
        t = x
        if not t.is_cuda:
            t = t.to(_device())
    else:
        t = torch.from_numpy(np.ascontiguousarray(x)).to(_device())
    if t.dtype != dtype:
        if dtype == torch.float64 and t.is_complex():
            raise ValueError("real signal carries complex values")
        t = t.to(dtype)
    return t.contiguous()


def _is_complex(x) -> bool:
    if isinstance(x, torch.Tensor):
        return x.is_complex()
    return np.iscomplexobj(x)


def _shape(x):
    return tuple(x.shape)


@dataclass(frozen=True)
class SphereGrid:
    """theta_t = pi(2t+1)/(2L-1), phi_p = 2 pi p/(2L-1) (sphere.py:41-63)."""

    band_limit: int

    def __post_init__(self):
        if self.band_limit < 1:
            raise ValueError(f"band limit must be positive, got {self.band_limit}")

    @cached_property
    def thetas(self) -> np.ndarray:
        L = self.band_limit
        return math.pi * (2.0 * np.arange(L) + 1.0) / (2 * L - 1)

    @cached_property
    def phis(self) -> np.ndarray:
        L = self.band_limit
        return 2.0 * math.pi * np.arange(2 * L - 1) / (2 * L - 1)

    @property
    def shape(self):
        return (self.band_limit, 2 * self.band_limit - 1)


@dataclass
class SphereSignal:
    """(L, 2L-1) theta-major samples of a spin-s field (sphere.py:66-90)."""

    grid: SphereGrid
    spin: int
    values: torch.Tensor
    real: bool = False

    def __post_init__(self):
        if _shape(self.values) != self.grid.shape:
            raise ValueError(f"values shape {_shape(self.values)} does not match grid {self.grid.shape}")
        if self.real:
            if self.spin != 0:
                raise ValueError("real signals must have spin 0")
            if _is_complex(self.values):
                raise ValueError("real signal carries complex values")
            self.values = as_device(self.values, torch.float64)
        else:
            self.values = as_device(self.values, torch.complex128)


@dataclass
class HarmonicCoeffs:
    """Flat f_lm at ell^2+ell+m; degrees below |spin| exactly zero
    (sphere.py:92-130)."""

    band_limit: int
    spin: int
    values: torch.Tensor
    real: bool = False
    # internal: set by this package's own producers (the forward SHT, the
    # synthesis accumulator after finish_acc), whose degrees below |spin| are
    # zero by construction, so the data-dependent check -- a host sync -- is
    # only paid for user-supplied coefficients
    trusted: bool = field(default=False, repr=False, compare=False, kw_only=True)

    def __post_init__(self):
        L = self.band_limit
        if L < 1:
            raise ValueError(f"band limit must be positive, got {L}")
        if abs(self.spin) >= L:
            raise ValueError(f"spin {self.spin} out of range for band limit {L}")
        self.values = as_device(self.values, torch.complex128)
        if _shape(self.values) != (L * L,):
            raise ValueError(f"expected {L * L} coefficients, got shape {_shape(self.values)}")
        low = self.spin * self.spin
        # a data-dependent check syncs the host: skipped for trusted producers
        # and while a CUDA graph is being captured (GraphedRoundTrip)
        if (low and not self.trusted and not torch.cuda.is_current_stream_capturing()
                and bool(torch.any(self.values[:low] != 0))):
            raise ValueError("degrees below |spin| must be exactly zero")
        if self.real and self.spin != 0:
            raise ValueError("real coefficient sets must have spin 0")

    def at(self, ell: int, m: int) -> complex:
        if not (0 <= ell < self.band_limit and abs(m) <= ell):
            raise ValueError(f"({ell}, {m}) out of range")
        return complex(self.values[lm_index(ell, m)].item())

    def degree_slice(self, ell: int) -> torch.Tensor:
        return self.values[ell * ell: ell * ell + 2 * ell + 1]


def _cdbl(t: torch.Tensor):
    return _cabi.ptr(t)


def sht_forward(f: SphereSignal) -> HarmonicCoeffs:
    """Forward spin SHT, exact for band-limited input (sphere.py:155-182)."""
    L = f.grid.band_limit
    s = f.spin
    if abs(s) >= L:
        raise ValueError(f"spin {s} out of range for band limit {L}")
    if f.real:
        return sht_forward_real(f)
    ctx = _cabi.context(f.values.device)
    out = torch.empty(L * L, dtype=torch.complex128, device=f.values.device)
    ctx.call("sht_forward", L, s, 0, _cdbl(f.values), _cdbl(out))
    return HarmonicCoeffs(L, s, out, trusted=True)


def sht_inverse(flm: HarmonicCoeffs) -> SphereSignal:
    """Evaluate coefficients on the MW grid (sphere.py:185-207)."""
    if flm.real:
        return sht_inverse_real(flm)
    L, s = flm.band_limit, flm.spin
    ctx = _cabi.context(flm.values.device)
    out = torch.empty((L, 2 * L - 1), dtype=torch.complex128, device=flm.values.device)
    ctx.call("sht_inverse", L, s, 0, _cdbl(flm.values), _cdbl(out))
    return SphereSignal(SphereGrid(L), s, out)


def sht_forward_real(f: SphereSignal) -> HarmonicCoeffs:
    """Real spin-0 forward via half spectra (sphere.py:210-236)."""
    if not f.real:
        raise ValueError("sht_forward_real requires a real-flagged signal")
    L = f.grid.band_limit
    ctx = _cabi.context(f.values.device)
    out = torch.empty(L * L, dtype=torch.complex128, device=f.values.device)
    ctx.call("sht_forward", L, 0, 1, _cdbl(f.values), _cdbl(out))
    return HarmonicCoeffs(L, 0, out, real=True, trusted=True)


def sht_inverse_real(flm: HarmonicCoeffs) -> SphereSignal:
    """Real-symmetric coefficients to real samples (sphere.py:239-260)."""
    if not flm.real:
        raise ValueError("sht_inverse_real requires real-flagged coefficients")
    L = flm.band_limit
    ctx = _cabi.context(flm.values.device)
    out = torch.empty((L, 2 * L - 1), dtype=torch.float64, device=flm.values.device)
    ctx.call("sht_inverse", L, 0, 1, _cdbl(flm.values), _cdbl(out))
    return SphereSignal(SphereGrid(L), 0, out, real=True)
