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
    """Our build_tiling (independent tanh-sinh quadrature of k_lambda) against
    the reference's own tilings.  The reference integrates k_lambda by Simpson
    panel doubling to tol = 1e-12 (tiling.py:74-148), so the squared profiles
    kappa_j^2 = k_outer - k_inner and Phi^2 agree to that level; kappa_j itself
    is their square root, which amplifies the reference's 1e-12 error to
    ~1e-6 absolute where kappa_j^2 is ~1e-12 (the band edges), so it is
    compared relatively where kappa_j^2 >= 1e-2."""
    from conftest import reference_tiling
    ref = reference_tiling(L, s, lam, j0)
    t = T.build_tiling(T.TilingParams(L, s, lam, j0))
    key = f"tiling_{L}_{s}_{lam}_{j0}"
    assert t.params.j_max == int(golden[key + "_jmax"]) == ref.params.j_max
    np.testing.assert_array_equal(ref.kernels, golden[key + "_kernels"])  # the recording is the fixture
    np.testing.assert_allclose(t.kernels ** 2, ref.kernels ** 2, rtol=0, atol=1e-11)
    np.testing.assert_allclose((t.scaling / np.sqrt((2 * np.arange(L) + 1) / (4 * math.pi))) ** 2,
                               (ref.scaling / np.sqrt((2 * np.arange(L) + 1) / (4 * math.pi))) ** 2, rtol=0, atol=1e-11)
    big = ref.kernels ** 2 >= 1e-2
    np.testing.assert_allclose(t.kernels[big], ref.kernels[big], rtol=1e-9, atol=0)
    np.testing.assert_array_equal(t.direction_pos, golden[key + "_dirpos"])
    np.testing.assert_array_equal(t.direction_neg, golden[key + "_dirneg"])
    np.testing.assert_allclose(t.angles, golden[key + "_angles"], rtol=0, atol=1e-15)
    pos, neg = T.curvelet_harmonics(t, t.params.j_max)
    rpos, rneg = T.curvelet_harmonics(ref, ref.params.j_max)
    np.testing.assert_array_equal(rpos, golden[key + "_psipos_jmax"])
    np.testing.assert_array_equal(rneg, golden[key + "_psineg_jmax"])
    amp2 = (2 * np.arange(L) + 1) / (8 * math.pi ** 2)
    np.testing.assert_allclose(pos ** 2 / amp2, rpos ** 2 / amp2, rtol=0, atol=1e-11)
    assert T.admissibility_residual(t) <= 1e-14
    assert T.admissibility_residual(ref) <= 1e-8


def test_step_against_adaptive_gauss_kronrod():
    """k_lambda from the tanh-sinh rule against scipy's adaptive Gauss-Kronrod
    (QUADPACK) at tight tolerance: an independent check of the quadrature."""
    from scipy import integrate
    for lam in (1.5, 2.0, 2.5, 3.0):
        def g(u):
            x = (2 * lam / (lam - 1)) * (math.exp(u) - 1 / lam) - 1
            return math.exp(-2 / (1 - x * x)) if abs(x) < 1 else 0.0
        den = integrate.quad(g, -math.log(lam), 0.0, epsabs=1e-17, epsrel=1e-14, limit=200)[0]
        for t in np.linspace(1 / lam + 1e-3, 1 - 1e-3, 9):
            ref = integrate.quad(g, math.log(t), 0.0, epsabs=1e-17, epsrel=1e-14, limit=200)[0] / den
            assert abs(T.smooth_step_k(lam, t) - ref) <= 1e-14, (lam, t)


def test_step_is_history_free():
    """k_lambda(t) does not depend on earlier queries (no memo table)."""
    a = T.smooth_step_k(2.0, 0.731)
    for t in np.linspace(0.5, 1.0, 37):
        T.smooth_step_k(2.0, t)
    T.build_tiling(T.TilingParams(1024, 0, 2.0, 3))
    assert T.smooth_step_k(2.0, 0.731) == a


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
