"""Delta(pi/2) table access (device-built, symmetry-reduced).

The reference tabulates full planes d^l_{m'm}(pi/2) on the host
(wigner.py:191-240).  Here the table is built on the GPU by the same
degree recursion (csrc/delta.cu) and stored as the 1/8 wedge
0 <= m <= m' <= l; ``halfpi_wedge`` returns it and ``wedge_index`` /
``wedge_value`` expand entries through the symmetries
    D_{-m',m} = (-1)^{l+m} D_{m'm},  D_{m',-m} = (-1)^{l+m'} D_{m'm},
    D_{m'm} = (-1)^{m'-m} D_{mm'}.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _cabi

__all__ = ["halfpi_wedge", "wedge_index", "wedge_plane", "wigner_d_edge_columns", "edge_column_table"]


def wedge_size(L: int) -> int:
    return L * (L + 1) * (L + 2) // 6


def wedge_index(l: int, mp: int, m: int):
    """(flat index, sign) of Delta^l_{mp,m} in the wedge layout."""
    neg = 0
    if mp < 0:
        mp = -mp
        neg ^= (l + m) & 1
    if m < 0:
        m = -m
        neg ^= (l + mp) & 1
    if mp < m:
        mp, m = m, mp
        neg ^= (mp - m) & 1
    return l * (l + 1) * (l + 2) // 6 + mp * (mp + 1) // 2 + m, (-1.0 if neg else 1.0)


def wedge_plane(wedge: np.ndarray, l: int) -> np.ndarray:
    """Expand plane l (rows m'+l, cols m+l) from a host copy of the wedge."""
    n = 2 * l + 1
    out = np.empty((n, n))
    for i in range(n):
        for j in range(n):
            k, s = wedge_index(l, i - l, j - l)
            out[i, j] = s * wedge[k]
    return out


def halfpi_wedge(L: int, device=None) -> torch.Tensor:
    """The device wedge table for l < L (float64, length L(L+1)(L+2)/6)."""
    if L < 1:
        raise ValueError(f"band limit must be positive, got {L}")
    ctx = _cabi.context(device)
    out = torch.empty(wedge_size(L), dtype=torch.float64, device=torch.device("cuda", ctx.device))
    ctx.call("halfpi_wedge", L, _cabi.ptr(out))
    return out


def edge_column_table(L: int, beta: float, device=None) -> torch.Tensor:
    """(L, 2L-1, 2) float64 device table: [l, k+L-1] = (d^l_{k,+l}(beta),
    d^l_{k,-l}(beta)) for |k| <= l, zero elsewhere (csrc/rotate.cu)."""
    if L < 1:
        raise ValueError(f"band limit must be positive, got {L}")
    ctx = _cabi.context(device)
    out = torch.empty((L, 2 * L - 1, 2), dtype=torch.float64, device=torch.device("cuda", ctx.device))
    ctx.call("edge_columns", L, float(beta), _cabi.ptr(out))
    return out


def wigner_d_edge_columns(ell: int, beta: float):
    """Columns d^ell_{k,+ell}(beta) and d^ell_{k,-ell}(beta) over k in
    [-ell, ell] (wigner.py:304-322), log-space closed forms on the device."""
    if ell < 0:
        raise ValueError(f"degree must be non-negative, got {ell}")
    tab = edge_column_table(ell + 1, beta)[ell]
    return tab[:, 0], tab[:, 1]
