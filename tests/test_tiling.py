"""Host tiling (kernel generation) against the reference's own outputs."""

import math

import numpy as np
import pytest

from paper_1511_05578_b200 import tiling as T
from paper_1511_05578_b200.transform import scale_band_limit, scaling_band_limit

CASES = [(64, 0, 2.0, 2), (128, 2, 2.0, 2), (512, 0, 2.0, 2), (1024, 0, 2.0, 3), (16, 0, 3.0, 0),
         (33, 1, 2.5, 1)]


@pytest.mark.parametrize("L,s,lam,j0", CASES)
def test_tiling_matches_reference(golden, L, s, lam, j0):
    from conftest import golden_tilings
    t = golden_tilings()[(L, s, lam, j0)]
    key = f"tiling_{L}_{s}_{lam}_{j0}"
    assert t.params.j_max == int(golden[key + "_jmax"])
    np.testing.assert_allclose(t.kernels, golden[key + "_kernels"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(t.scaling, golden[key + "_scaling"], rtol=0, atol=1e-12)
    np.testing.assert_array_equal(t.direction_pos, golden[key + "_dirpos"])
    np.testing.assert_array_equal(t.direction_neg, golden[key + "_dirneg"])
    np.testing.assert_allclose(t.angles, golden[key + "_angles"], rtol=0, atol=1e-15)
    pos, neg = T.curvelet_harmonics(t, t.params.j_max)
    np.testing.assert_allclose(pos, golden[key + "_psipos_jmax"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(neg, golden[key + "_psineg_jmax"], rtol=0, atol=1e-12)
    assert T.admissibility_residual(t) <= 1e-8


def test_params_validation():
    with pytest.raises(ValueError):
        T.TilingParams(0)
    with pytest.raises(ValueError):
        T.TilingParams(16, lam=1.0)
    with pytest.raises(ValueError):
        T.TilingParams(16, j_min=-1)
    with pytest.raises(ValueError):
        T.TilingParams(16, j_min=5, j_max=3)
    with pytest.raises(ValueError):
        T.TilingParams(4, 0, 3.0, 2)  # scale range collapses (tests/test_transform.py:128-131)
    with pytest.raises(ValueError):
        T.build_tiling(T.TilingParams(16), tol=0.0)


def test_band_limits_and_bump():
    p = T.TilingParams(128, 0, 2.0, 2)
    assert scale_band_limit(p, 2) == 8 and scale_band_limit(p, 6) == 128 and scale_band_limit(p, 7) == 128
    assert scaling_band_limit(p) == 4
    with pytest.raises(ValueError):
        scale_band_limit(p, 1)
    assert T.schwartz_s(0.0) == pytest.approx(math.exp(-1.0))
    assert T.schwartz_s(1.0) == 0.0
    assert T.smooth_step_k(2.0, 0.5) == 1.0 and T.smooth_step_k(2.0, 1.0) == 0.0
    assert 0.0 < T.smooth_step_k(2.0, 0.75) < 1.0
