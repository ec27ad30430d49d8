"""SO(3) containers and the curvelet-sparse Wigner transforms (device).

Drop-in mirror of the curvelet part of ``scurve.so3`` (so3.py:45-182,
214-285, 349-417): ``SO3Grid``, ``SO3Signal``, ``CurveletWignerCoeffs``,
``so3_inverse_curvelet(_real)`` and ``so3_forward_curvelet(_real)`` with
the same shapes, ValueError/TypeError conditions and layouts.  The dense
O(L^4) "general" transforms are validation oracles in the reference and
are out of scope here.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import cached_property

import numpy as np
import torch

from . import _cabi
from .sphere import _is_complex, _shape, as_device

__all__ = [
    "CurveletWignerCoeffs",
    "SO3Grid",
    "SO3Signal",
    "SO3Slab",
    "WignerCoeffs",
    "so3_forward_curvelet",
    "so3_forward_curvelet_slab",
    "so3_forward_curvelet_real",
    "so3_inverse_curvelet",
    "so3_inverse_curvelet_real",
    "so3_inverse_curvelet_slab",
    "so3_forward_general",
    "so3_inverse_general",
]


@dataclass(frozen=True)
class SO3Grid:
    """L betas, 2M-1 alphas, 2N-1 gammas; shape (2N-1, L, 2M-1) (so3.py:45-72)."""

    L: int
    M: int
    N: int

    def __post_init__(self):
        for name in ("L", "M", "N"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be positive, got {getattr(self, name)}")

    @cached_property
    def alphas(self) -> np.ndarray:
        return 2.0 * math.pi * np.arange(2 * self.M - 1) / (2 * self.M - 1)

    @cached_property
    def betas(self) -> np.ndarray:
        return math.pi * (2.0 * np.arange(self.L) + 1.0) / (2 * self.L - 1)

    @cached_property
    def gammas(self) -> np.ndarray:
        return 2.0 * math.pi * np.arange(2 * self.N - 1) / (2 * self.N - 1)

    @property
    def shape(self):
        return (2 * self.N - 1, self.L, 2 * self.M - 1)


@dataclass
class SO3Signal:
    """(gamma, beta, alpha) samples (so3.py:75-90)."""

    grid: SO3Grid
    values: torch.Tensor
    real: bool = False

    def __post_init__(self):
        if _shape(self.values) != self.grid.shape:
            raise ValueError(f"values shape {_shape(self.values)} does not match grid {self.grid.shape}")
        if self.real and _is_complex(self.values):
            raise ValueError("real signal carries complex values")
        self.values = as_device(self.values, torch.float64 if self.real else torch.complex128)


@dataclass
class CurveletWignerCoeffs:
    """Outer columns n=+-ell: values (2, L, 2L-1) (so3.py:124-182)."""

    band_limit: int
    values: torch.Tensor

    def __post_init__(self):
        L = self.band_limit
        if L < 1:
            raise ValueError(f"band limit must be positive, got {L}")
        self.values = as_device(self.values, torch.complex128)
        if _shape(self.values) != (2, L, 2 * L - 1):
            raise ValueError(f"expected shape {(2, L, 2 * L - 1)}, got {_shape(self.values)}")

    @classmethod
    def zeros(cls, L: int) -> "CurveletWignerCoeffs":
        return cls(L, np.zeros((2, L, 2 * L - 1), complex))

    def row(self, n: int) -> torch.Tensor:
        ell = abs(n)
        if ell >= self.band_limit:
            raise ValueError(f"|n| = {ell} out of range")
        c = self.band_limit - 1
        return self.values[0 if n >= 0 else 1, ell, c - ell: c + ell + 1]

    def set_row(self, n: int, row) -> None:
        self.row(n)[:] = as_device(row, torch.complex128)

    def densify(self) -> "WignerCoeffs":
        """Dense coefficients holding the outer columns n = +-ell (so3.py:176-182)."""
        return densify(self)


def plane_offset(ell: int) -> int:
    """Start of plane ell in the packed dense layout: sum_{l<ell} (2l+1)^2."""
    return ell * (4 * ell * ell - 1) // 3


class WignerCoeffs:
    """Dense Wigner coefficients: planes[ell][m + ell, n + ell] (so3.py:93-121).

    The planes live packed back to back in one device tensor ``values``
    (plane ell at ``plane_offset(ell)``, L(4L^2-1)/3 complex128 entries);
    ``planes`` is the reference's list of (2l+1, 2l+1) views into it.
    """

    def __init__(self, band_limit: int, planes=None, *, values=None):
        L = int(band_limit)
        if L < 1:
            raise ValueError(f"band limit must be positive, got {L}")
        self.band_limit = L
        if values is not None:
            v = as_device(values, torch.complex128).reshape(-1)
            if v.numel() != plane_offset(L):
                raise ValueError(f"expected {plane_offset(L)} packed entries, got {v.numel()}")
            self.values = v
        else:
            if planes is None or len(planes) != L:
                raise ValueError(f"expected {L} planes, got {0 if planes is None else len(planes)}")
            for ell, pl in enumerate(planes):
                if _shape(pl) != (2 * ell + 1, 2 * ell + 1):
                    raise ValueError(f"plane {ell} has shape {_shape(pl)}")
            self.values = torch.cat([as_device(pl, torch.complex128).reshape(-1) for pl in planes])

    @property
    def planes(self) -> list:
        return [self.plane(ell) for ell in range(self.band_limit)]

    def plane(self, ell: int) -> torch.Tensor:
        if not 0 <= ell < self.band_limit:
            raise ValueError(f"degree {ell} out of range")
        n = 2 * ell + 1
        return self.values[plane_offset(ell): plane_offset(ell + 1)].view(n, n)

    @classmethod
    def zeros(cls, L: int) -> "WignerCoeffs":
        if L < 1:
            raise ValueError(f"band limit must be positive, got {L}")
        return cls(L, values=torch.zeros(plane_offset(L), dtype=torch.complex128, device=_dev()))

    @classmethod
    def random(cls, L: int, rng: np.random.Generator) -> "WignerCoeffs":
        planes = [rng.uniform(-1, 1, (2 * ell + 1, 2 * ell + 1))
                  + 1j * rng.uniform(-1, 1, (2 * ell + 1, 2 * ell + 1)) for ell in range(L)]
        return cls(L, planes)


def _dev():
    from .sphere import _device
    return _device()


def _check_sparse_grid(w, grid):
    if not isinstance(w, CurveletWignerCoeffs):
        raise TypeError("sparse synthesis requires CurveletWignerCoeffs")
    L = w.band_limit
    if not (grid.L == L and grid.M == L and grid.N == L):
        raise ValueError("sparse path requires a grid with N = M = L matching the coefficients")
    return L


def so3_inverse_curvelet(w: CurveletWignerCoeffs, grid: SO3Grid, out: torch.Tensor | None = None) -> SO3Signal:
    """Sparse synthesis onto the grid, O(L^3 log L) (so3.py:259-285)."""
    L = _check_sparse_grid(w, grid)
    K = 2 * L - 1
    dev = w.values.device
    if out is None:
        out = torch.empty((K, L, K), dtype=torch.complex128, device=dev)
    _cabi.checked(out, torch.complex128, (K, L, K), dev, "out")
    _cabi.context(dev).call("so3_inverse_curvelet", L, 0, _cabi.ptr(w.values), _cabi.ptr(out))
    return SO3Signal(grid, out)


def so3_inverse_curvelet_real(w: CurveletWignerCoeffs, grid: SO3Grid, out: torch.Tensor | None = None) -> SO3Signal:
    """Sparse synthesis to real samples via half the gamma spectrum
    (so3.py:386-417); assumes real-signal symmetry of the coefficients."""
    L = _check_sparse_grid(w, grid)
    K = 2 * L - 1
    dev = w.values.device
    if out is None:
        out = torch.empty((K, L, K), dtype=torch.float64, device=dev)
    _cabi.checked(out, torch.float64, (K, L, K), dev, "out")
    _cabi.context(dev).call("so3_inverse_curvelet", L, 1, _cabi.ptr(w.values), _cabi.ptr(out))
    return SO3Signal(grid, out, real=True)


def _check_forward(f: SO3Signal) -> int:
    grid = f.grid
    L = grid.L
    if not (grid.M == L and grid.N == L):
        raise ValueError("sparse path requires N = M = L")
    return L


def so3_forward_curvelet(f: SO3Signal, out: torch.Tensor | None = None) -> CurveletWignerCoeffs:
    """Forward Wigner transform onto the n=+-ell columns (so3.py:214-244)."""
    L = _check_forward(f)
    vals = f.values if not f.real else f.values.to(torch.complex128)
    dev = vals.device
    if out is None:
        out = torch.empty((2, L, 2 * L - 1), dtype=torch.complex128, device=dev)
    _cabi.checked(out, torch.complex128, (2, L, 2 * L - 1), dev, "out")
    _cabi.checked(vals, torch.complex128, (2 * L - 1, L, 2 * L - 1), dev, "signal values")
    _cabi.context(dev).call("so3_forward_curvelet", L, 0, _cabi.ptr(vals), _cabi.ptr(out))
    return CurveletWignerCoeffs(L, out)


def so3_forward_curvelet_real(f: SO3Signal, out: torch.Tensor | None = None) -> CurveletWignerCoeffs:
    """Forward transform of a real signal via rfft along gamma (so3.py:349-383)."""
    if not f.real:
        raise ValueError("real path requires a real-flagged signal")
    L = _check_forward(f)
    dev = f.values.device
    if out is None:
        out = torch.empty((2, L, 2 * L - 1), dtype=torch.complex128, device=dev)
    _cabi.checked(out, torch.complex128, (2, L, 2 * L - 1), dev, "out")
    _cabi.checked(f.values, torch.float64, (2 * L - 1, L, 2 * L - 1), dev, "signal values")
    _cabi.context(dev).call("so3_forward_curvelet", L, 1, _cabi.ptr(f.values), _cabi.ptr(out))
    return CurveletWignerCoeffs(L, out)


# ---------------------------------------------------------------------------
# beta slabs (multi-GPU sharding of one scale)
# ---------------------------------------------------------------------------
@dataclass
class SO3Slab:
    """Beta rows [b0, b0 + nb) of an SO(3) signal on `grid`: values
    (2N-1, nb, 2M-1) = the full signal's values[:, b0:b0+nb, :]."""

    grid: SO3Grid
    b0: int
    values: torch.Tensor
    real: bool = False

    @property
    def nb(self) -> int:
        return int(self.values.shape[1])

    def __post_init__(self):
        K_g, _, K_a = self.grid.shape
        if self.real and _is_complex(self.values):
            raise ValueError("real slab carries complex values")
        # a view such as full.values[:, b0:b0+nb, :] is not contiguous: copy it
        # into the dense (K, nb, K) layout the C ABI reads
        self.values = as_device(self.values, torch.float64 if self.real else torch.complex128)
        if self.b0 < 0 or self.values.dim() != 3 or self.b0 + self.values.shape[1] > self.grid.L:
            raise ValueError(f"slab rows [{self.b0}, {self.b0 + self.values.shape[1]}) outside [0, {self.grid.L})")
        if (self.values.shape[0], self.values.shape[2]) != (K_g, K_a):
            raise ValueError(f"slab shape {tuple(self.values.shape)} does not match grid {self.grid.shape}")


def so3_inverse_curvelet_slab(w: CurveletWignerCoeffs, grid: SO3Grid, b0: int, nb: int,
                              out: torch.Tensor | None = None) -> SO3Slab:
    """Rows [b0, b0+nb) of so3_inverse_curvelet(w, grid) (complex path)."""
    L = _check_sparse_grid(w, grid)
    K = 2 * L - 1
    dev = w.values.device
    if out is None:
        out = torch.empty((K, nb, K), dtype=torch.complex128, device=dev)
    _cabi.checked(out, torch.complex128, (K, nb, K), dev, "out")
    _cabi.context(dev).call("so3_inverse_curvelet_slab", L, _cabi.ptr(w.values), int(b0), int(nb), _cabi.ptr(out))
    return SO3Slab(grid, int(b0), out)


def so3_forward_curvelet_slab(f: SO3Slab, out: torch.Tensor | None = None, accumulate: bool = False) -> CurveletWignerCoeffs:
    """The slab's partial sum of so3_forward_curvelet(_real): summed over all
    slabs of a signal it equals the full forward transform (so3.py:203-243)."""
    L = _check_forward(f)
    dev = f.values.device
    if out is None:
        out = torch.zeros((2, L, 2 * L - 1), dtype=torch.complex128, device=dev)
        accumulate = False
    _cabi.checked(out, torch.complex128, (2, L, 2 * L - 1), dev, "out")
    K = 2 * L - 1
    _cabi.checked(f.values, torch.float64 if f.real else torch.complex128, (K, f.nb, K), dev, "slab values")
    _cabi.context(dev).call("so3_forward_curvelet_slab", L, 1 if f.real else 0, _cabi.ptr(f.values), int(f.b0),
                            f.nb, _cabi.ptr(out), 1 if accumulate else 0)
    return CurveletWignerCoeffs(L, out)


def so3_inverse_general(w: WignerCoeffs, grid: SO3Grid) -> SO3Signal:
    """Dense synthesis onto the grid, O(L^4) (so3.py:317-346): the reference's
    cross-check of the curvelet-sparse path, on the device (csrc/general.cu)."""
    if isinstance(w, CurveletWignerCoeffs):
        raise TypeError("dense synthesis requires WignerCoeffs; use densify() first")
    if not isinstance(w, WignerCoeffs):
        raise TypeError("dense synthesis requires WignerCoeffs")
    L = w.band_limit
    if L > min(grid.L, grid.M, grid.N):
        raise ValueError(f"band limit {L} exceeds grid {grid}")
    ctx = _cabi.context(w.values.device)
    out = torch.empty(grid.shape, dtype=torch.complex128, device=w.values.device)
    ctx.call("so3_inverse_general", L, grid.L, grid.M, grid.N, _cabi.ptr(w.values), _cabi.ptr(out))
    return SO3Signal(grid, out)


def densify(w: CurveletWignerCoeffs) -> WignerCoeffs:
    """Dense coefficients holding only the outer columns n = +-ell of `w`."""
    if not isinstance(w, CurveletWignerCoeffs):
        raise TypeError("densify expects sparse coefficients")
    L = w.band_limit
    d = WignerCoeffs.zeros(L)
    c = L - 1
    for ell in range(L):
        pl = d.plane(ell)
        pl[:, 2 * ell] = w.values[0, ell, c - ell: c + ell + 1]
        if ell > 0:
            pl[:, 0] = w.values[1, ell, c - ell: c + ell + 1]
    return d


def so3_forward_general(f: SO3Signal, band_limit: int | None = None) -> WignerCoeffs:
    """Dense forward Wigner transform, O(L^4) (so3.py:288-314), on the device:
    the (gamma, alpha) spectrum by cuFFT, then direct beta and Delta sums."""
    grid = f.grid
    L = grid.L if band_limit is None else int(band_limit)
    if L > min(grid.L, grid.M, grid.N):
        raise ValueError(f"band limit {L} exceeds grid {grid}")
    if f.real:
        raise ValueError("dense forward transform takes complex samples")
    ctx = _cabi.context(f.values.device)
    out = WignerCoeffs(L, values=torch.empty(plane_offset(L), dtype=torch.complex128, device=f.values.device))
    ctx.call("so3_forward_general", L, grid.L, grid.M, grid.N, _cabi.ptr(f.values), _cabi.ptr(out.values))
    return out
