"""Pin the CPU oracle against the reference's own outputs (golden fixtures).

The fixtures come from the unmodified reference package
(tests/golden/make_golden.py).  Tolerances: the restatement follows the
same arithmetic, so agreement is near machine precision.
"""

import math

import numpy as np
import pytest

from oracle import scurve_oracle as orc


def test_halfpi_small_table(golden):
    flat = np.concatenate([p.ravel() for p in orc.halfpi_planes(12)])
    np.testing.assert_allclose(flat, golden["halfpi_L12"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("ell", [33, 64, 65])
def test_halfpi_large_planes(golden, ell):
    planes = orc.halfpi_planes(ell + 1)
    np.testing.assert_allclose(planes[ell], golden[f"halfpi_plane_{ell}"], rtol=0, atol=1e-15)


def test_halfpi_exact_kat(golden):
    planes = orc.halfpi_planes(33)
    for ell, mp, m, val in golden["halfpi_kat"]:
        ell, mp, m = int(ell), int(mp), int(m)
        assert abs(planes[ell][mp + ell, m + ell] - val) <= 1e-12


def test_halfpi_frozen_values():
    planes = orc.halfpi_planes(3)
    assert planes[2][4, 4] == pytest.approx(0.25, abs=1e-15)
    np.testing.assert_allclose(planes[1], [[0.5, 1 / math.sqrt(2), 0.5],
                                           [-1 / math.sqrt(2), 0, 1 / math.sqrt(2)],
                                           [0.5, -1 / math.sqrt(2), 0.5]])


def test_weights(golden):
    np.testing.assert_array_equal(orc.weight_kernel(14), golden["weight_kernel_7"])
    w = orc.weight_kernel(4)
    assert w[4] == 2 and w[5] == 0.5j * math.pi and w[3] == -0.5j * math.pi
    assert w[6] == pytest.approx(-2 / 3) and w[7] == 0


@pytest.mark.parametrize("L", [1, 2, 3, 8, 16])
def test_weighted_convolve(golden, L):
    x = golden[f"wconv_in_{L}"]
    got = orc.weighted_convolve(x, axis=0)
    np.testing.assert_allclose(got, golden[f"wconv_out_{L}"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(orc.weighted_convolve_direct(x), got, rtol=0, atol=1e-11)


@pytest.mark.parametrize("L,s", [(8, 0), (8, 2), (16, 1), (33, 0)])
def test_sht(golden, L, s):
    flm = golden[f"sht_flm_{L}_{s}"]
    f = orc.sht_inverse(flm, L, s)
    assert orc.rel_err(f, golden[f"sht_map_{L}_{s}"]) <= 1e-13
    back = orc.sht_forward(golden[f"sht_map_{L}_{s}"], L, s)
    assert orc.rel_err(back, golden[f"sht_fwd_{L}_{s}"]) <= 1e-13
    raw = orc.sht_forward(golden[f"sht_rawmap_{L}_{s}"], L, s)
    assert orc.rel_err(raw, golden[f"sht_rawfwd_{L}_{s}"]) <= 1e-13


@pytest.mark.parametrize("L", [8, 17])
def test_sht_real(golden, L):
    f = orc.sht_inverse_real(golden[f"shtr_flm_{L}"], L)
    assert orc.rel_err(f, golden[f"shtr_map_{L}"]) <= 1e-13
    back = orc.sht_forward_real(golden[f"shtr_map_{L}"], L)
    assert orc.rel_err(back, golden[f"shtr_fwd_{L}"]) <= 1e-13


@pytest.mark.parametrize("L", [4, 8, 13])
def test_so3_curvelet(golden, L):
    f = orc.so3_inverse_curvelet(golden[f"so3_w_{L}"])
    assert orc.rel_err(f, golden[f"so3_inv_{L}"]) <= 1e-13
    w = orc.so3_forward_curvelet(golden[f"so3_inv_{L}"])
    assert orc.rel_err(w, golden[f"so3_fwd_{L}"]) <= 1e-13
    raw = orc.so3_forward_curvelet(golden[f"so3_raw_{L}"])
    assert orc.rel_err(raw, golden[f"so3_rawfwd_{L}"]) <= 1e-13


@pytest.mark.parametrize("L", [5, 8])
def test_so3_curvelet_real(golden, L):
    f = orc.so3_inverse_curvelet_real(golden[f"so3r_w_{L}"])
    assert orc.rel_err(f, golden[f"so3r_inv_{L}"]) <= 1e-13
    w = orc.so3_forward_curvelet_real(golden[f"so3r_inv_{L}"])
    assert orc.rel_err(w, golden[f"so3r_fwd_{L}"]) <= 1e-13


# Transform fixtures are compared on the exact tiling arrays the reference
# used (tests/golden/reference_tilings.npz), so only the transform arithmetic
# is under test here.
TILING_TOL = 1e-12


def _psi_from_golden(golden, L, s, j_min, k=0):
    from conftest import reference_tiling
    from paper_1511_05578_b200 import tiling as T
    t = reference_tiling(L, s, 2.0, j_min, k)
    psi = [T.curvelet_harmonics(t, j) for j in range(j_min, t.params.j_max + 1)]
    return t, psi


@pytest.mark.parametrize("L,s,real", [(16, 0, False), (16, 2, False), (16, 0, True)])
def test_transform_small(golden, L, s, real):
    # the generator built (16, 0, 2, 2) twice: complex first, then real
    t, psi = _psi_from_golden(golden, L, s, 2, 1 if real else 0)
    key = f"xf_{L}_{s}_{int(real)}"
    f = golden[key + "_map"]
    smap, scales = orc.analyze(f, L, s, 2.0, 2, t.params.j_max, psi, t.scaling, real=real)
    assert orc.rel_err(smap, golden[key + "_scaling"]) <= TILING_TOL
    for i, sig in enumerate(scales):
        assert orc.rel_err(sig, golden[key + f"_scale{i}"]) <= TILING_TOL
    g = orc.synthesize(smap, scales, L, s, 2.0, 2, t.params.j_max, psi, t.scaling, real=real)
    assert orc.rel_err(g, golden[key + "_recon"]) <= TILING_TOL
    assert orc.rel_err(g, f) <= 1e-11


def test_config1_L64(golden):
    L = 64
    t, psi = _psi_from_golden(golden, L, 0, 2, 1)  # after tiling_cases' (64, 0, 2, 2)
    f = golden["c1_map"]
    flm = orc.gaussian_flm(L, 0, 0, real=True)
    assert orc.rel_err(orc.sht_inverse(flm, L, 0), f) <= 1e-13
    smap, scales = orc.analyze(f, L, 0, 2.0, 2, t.params.j_max, psi, t.scaling)
    assert orc.rel_err(smap, golden["c1_scaling"]) <= TILING_TOL
    for i, sig in enumerate(scales):
        idx = golden[f"c1_scale{i}_idx"]
        assert orc.rel_err(sig[tuple(idx.T)], golden[f"c1_scale{i}_val"]) <= TILING_TOL
        assert abs(sig.sum() - golden[f"c1_scale{i}_sum"]) <= 1e-9 * golden[f"c1_scale{i}_l2"]
    g = orc.synthesize(smap, scales, L, 0, 2.0, 2, t.params.j_max, psi, t.scaling)
    assert orc.rel_err(g, golden["c1_recon"]) <= TILING_TOL
    w = orc.so3_forward_curvelet(scales[-1])
    assert orc.rel_err(w, golden["c1_wlast"]) <= TILING_TOL


@pytest.mark.parametrize("L", [8, 16, 24, 64])
def test_beta_row_restatement_matches_full_oracle(L):
    """The per-beta-row oracle used for the full-size (L=1024, 2048) GPU checks
    restates the same linear map as the full so3_inverse_curvelet oracle
    (itself pinned to the reference goldens above)."""
    rng = np.random.default_rng(L)
    K = 2 * L - 1
    w = rng.standard_normal((2, L, K)) + 1j * rng.standard_normal((2, L, K))
    full = orc.so3_inverse_curvelet(w)
    for b in (0, L // 2, L - 1):
        assert orc.rel_err(orc.so3_inverse_curvelet_beta_row(w, b), full[:, b, :]) <= 1e-13
