"""Argument validation in front of the C ABI (CPU part): a raw pointer only
reaches the library after device, dtype, layout and shape are checked."""

import pytest
import torch

from paper_1511_05578_b200 import _cabi


def test_checked_rejects_bad_buffers_cpu():
    t = torch.zeros((3, 4), dtype=torch.complex128)
    with pytest.raises(TypeError):
        _cabi.checked(t.numpy(), torch.complex128, (3, 4), torch.device("cuda", 0))
    with pytest.raises(TypeError):
        _cabi.checked(t.real.contiguous(), torch.complex128, (3, 4), torch.device("cuda", 0))
    with pytest.raises(ValueError, match="must live on"):
        _cabi.checked(t, torch.complex128, (3, 4), torch.device("cuda", 0))


@pytest.mark.gpu
def test_out_buffers_are_validated_on_gpu():
    import paper_1511_05578_b200 as sc
    L = 8
    K = 2 * L - 1
    grid = sc.SO3Grid(L, L, L)
    w = sc.CurveletWignerCoeffs.zeros(L)
    with pytest.raises(TypeError):  # float64 where complex128 is written: would overrun
        sc.so3_inverse_curvelet(w, grid, out=torch.empty((K, L, K), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        sc.so3_inverse_curvelet(w, grid, out=torch.empty((K, L - 1, K), dtype=torch.complex128, device="cuda"))
    big = torch.empty((K, 2 * L, K), dtype=torch.complex128, device="cuda")
    with pytest.raises(ValueError, match="contiguous"):
        sc.so3_inverse_curvelet(w, grid, out=big[:, :L, :])
    f = sc.so3_inverse_curvelet(w, grid)
    with pytest.raises(ValueError):
        sc.so3_forward_curvelet(f, out=torch.empty((2, L, K + 2), dtype=torch.complex128, device="cuda"))


@pytest.mark.gpu
def test_slab_view_values_are_made_contiguous():
    """SO3Slab(values=full[:, b0:b0+nb, :]) -- a strided view -- is copied to
    the dense layout, so the slab forward reads the right rows."""
    import numpy as np
    import paper_1511_05578_b200 as sc
    from oracle import scurve_oracle as orc
    L = 128  # the slab entry points need the beta-quadrature path (128 <= L <= 2048)
    rng = np.random.default_rng(1)
    w = np.zeros((2, L, 2 * L - 1), complex)
    c = L - 1
    for l in range(L):
        for sh in range(2 if l else 1):
            w[sh, l, c - l:c + l + 1] = rng.standard_normal(2 * l + 1) + 1j * rng.standard_normal(2 * l + 1)
    grid = sc.SO3Grid(L, L, L)
    full = sc.so3_inverse_curvelet(sc.CurveletWignerCoeffs(L, w), grid)
    acc = None
    for b0, b1 in ((0, 40), (40, L)):
        slab = sc.SO3Slab(grid, b0, full.values[:, b0:b1, :])
        assert slab.values.is_contiguous()
        part = sc.so3_forward_curvelet_slab(slab, out=acc, accumulate=acc is not None)
        acc = part.values
    assert orc.rel_err(acc.cpu().numpy(), w) <= 1e-11
