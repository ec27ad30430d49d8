"""The reference's behavioural tests (tests/test_transform.py, tests/test_so3.py
of the reference package), restated on the device path: single-harmonic
localisation, multires = fullres, scaling-band support, coefficient energy,
constant signals, and the sparse transforms against the dense O(L^4) ones."""

import dataclasses
import math

import numpy as np
import pytest
import torch

from oracle import scurve_oracle as orc

pytestmark = pytest.mark.gpu


def _sc():
    import paper_1511_05578_b200 as sc
    return sc


def host(t):
    return t.detach().cpu().numpy()


def _random_flm(L, spin, rng, real=False):
    return orc.gaussian_flm(L, spin, seed=int(rng.integers(1 << 30)), real=real)


def test_single_harmonic_lands_on_one_scale():
    """test_transform.py:92-108."""
    sc = _sc()
    L, ell0, m0 = 8, 4, 1
    t = sc.build_tiling(sc.TilingParams(L, 0, 2.0, 0))
    vals = np.zeros(L * L, dtype=complex)
    vals[sc.lm_index(ell0, m0)] = 1.0
    c = sc.analyze(sc.sht_inverse(sc.HarmonicCoeffs(L, 0, vals)), t)
    pos, neg = sc.curvelet_harmonics(t, 2)
    w = sc.so3_forward_curvelet(c.scale(2))
    factor = 8 * math.pi ** 2 / (2 * ell0 + 1)
    assert abs(complex(w.row(ell0)[m0 + ell0]) - factor * pos[ell0]) <= 1e-12
    assert abs(complex(w.row(-ell0)[m0 + ell0]) - factor * neg[ell0]) <= 1e-12
    for j in (0, 1, 3):
        assert float(c.scale(j).values.abs().max()) <= 1e-13
    assert float(c.scaling.values.abs().max()) <= 1e-13


@pytest.mark.parametrize("L", [8, 16])
def test_multires_and_fullres_agree(L, rng):
    """test_transform.py:146-151, plus the full-resolution round trip."""
    sc = _sc()
    t = sc.build_tiling(sc.TilingParams(L, 0, 2.0, 0))
    f = sc.sht_inverse(sc.HarmonicCoeffs(L, 0, _random_flm(L, 0, rng)))
    a = sc.synthesize(sc.analyze(f, t, multires=True), t)
    cf = sc.analyze(f, t, multires=False)
    assert all(s.grid.L == L for s in cf.scales) and cf.scaling.grid.band_limit == L
    b = sc.synthesize(cf, t)
    assert float((a.values - b.values).abs().max()) <= 1e-10
    assert orc.rel_err(host(b.values), host(f.values)) <= 1e-11


def test_scaling_part_carries_only_coarse_degrees(rng):
    """test_transform.py:153-168."""
    sc = _sc()
    L, j_min = 16, 2
    t = sc.build_tiling(sc.TilingParams(L, 0, 2.0, j_min))
    vals = _random_flm(L, 0, rng)
    lam_pow = int(2 ** (j_min + 1))
    vals[: lam_pow * lam_pow] = 0.0
    flm = sc.HarmonicCoeffs(L, 0, vals)
    c = sc.analyze(sc.sht_inverse(flm), t)
    zero = sc.SphereSignal(c.scaling.grid, 0, torch.zeros_like(c.scaling.values))
    g = sc.synthesize(dataclasses.replace(c, scaling=zero), t)
    assert float((sc.sht_forward(g).values - flm.values).abs().max()) <= 1e-10


@pytest.mark.parametrize("L,spin", [(16, 0), (16, 2), (32, 1)])
def test_coefficient_energy_matches_signal_energy(L, spin, rng):
    """test_transform.py:183-195 (the frame's Parseval identity)."""
    sc = _sc()
    t = sc.build_tiling(sc.TilingParams(L, spin, 2.0, 1))
    flm = sc.HarmonicCoeffs(L, spin, _random_flm(L, spin, rng))
    c = sc.analyze(sc.sht_inverse(flm), t)
    total = float((sc.sht_forward(c.scaling).values.abs() ** 2).sum())
    for sig in c.scales:
        w = sc.so3_forward_curvelet(sig)
        for ell in range(1, w.band_limit):
            weight = (2 * ell + 1) / (8 * math.pi ** 2)
            total += weight * float((w.row(ell).abs() ** 2).sum() + (w.row(-ell).abs() ** 2).sum())
    expect = float((flm.values.abs() ** 2).sum())
    assert abs(total - expect) <= 1e-9 * expect


def test_constant_signal_is_scaling_only():
    """test_transform.py:342-351 (real path)."""
    sc = _sc()
    L = 16
    t = sc.build_tiling(sc.TilingParams(L, 0, 2.0, 2))
    g = sc.SphereGrid(L)
    f = sc.SphereSignal(g, 0, np.ones(g.shape), real=True)
    c = sc.analyze_real(f, t)
    for sig in c.scales:
        assert float(sig.values.abs().max()) <= 1e-13
    back = sc.synthesize_real(c, t)
    np.testing.assert_allclose(host(back.values), 1.0, atol=1e-12)


@pytest.mark.parametrize("L", [8, 16])
def test_sparse_transforms_match_general(L, rng):
    """test_so3.py inverse/forward_matches_general: the curvelet-sparse pair
    against the dense O(L^4) transforms on the outer columns."""
    sc = _sc()
    v = rng.uniform(-1, 1, (2, L, 2 * L - 1)) + 1j * rng.uniform(-1, 1, (2, L, 2 * L - 1))
    for ell in range(L):
        v[:, ell, : L - 1 - ell] = 0
        v[:, ell, L + ell:] = 0
    v[1, 0] = 0
    w = sc.CurveletWignerCoeffs(L, v)
    grid = sc.SO3Grid(L, L, L)
    sig = sc.so3_inverse_curvelet(w, grid)
    assert orc.rel_err(host(sig.values), host(sc.so3_inverse_general(w.densify(), grid).values)) <= 1e-12
    dense = sc.so3_forward_general(sig)
    fw = sc.so3_forward_curvelet(sig)
    for ell in range(L):
        col_p = host(dense.plane(ell)[:, 2 * ell])
        assert np.abs(col_p - host(fw.row(ell))).max() <= 1e-11
        if ell > 0:
            col_n = host(dense.plane(ell)[:, 0])
            assert np.abs(col_n - host(fw.row(-ell))).max() <= 1e-11


def test_single_entry_matches_general():
    """test_so3.py single_entry_matches_general: one nonzero coefficient."""
    sc = _sc()
    L = 8
    v = np.zeros((2, L, 2 * L - 1), complex)
    v[1, 5, (L - 1) + 3] = 0.7 - 0.2j
    w = sc.CurveletWignerCoeffs(L, v)
    grid = sc.SO3Grid(L, L, L)
    a = host(sc.so3_inverse_curvelet(w, grid).values)
    b = host(sc.so3_inverse_general(w.densify(), grid).values)
    assert np.abs(a - b).max() <= 1e-13
