"""Frame rotation: rotate_to_north / rotate_from_north
(reference transform.py:256-297) and wigner_d_edge_columns (wigner.py:304-322).

CPU tests pin the oracle restatement to fixtures made by the unmodified
reference (tests/golden/make_golden.py, reference_rotation.npz).  GPU tests
run the CUDA kernels (csrc/rotate.cu) through the C ABI against the same
fixtures, the live oracle, and the reference's own properties
(tests/test_transform.py:198-230): round trip, per-m energy, identity angle,
projection idempotence; and at L=1024 (the C4 finest scale) through
size-independent properties.
"""

import math
import os
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import scurve_oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rot():
    with np.load(os.path.join(ROOT, "tests", "golden", "reference_rotation.npz")) as z:
        return {k: z[k] for k in z.files}


def _t(theta):
    """Minimal tiling carrying one scale angle (only params.j_min/j_max and angles are read)."""
    return SimpleNamespace(params=SimpleNamespace(j_min=0, j_max=0), angles=np.array([float(theta)]))


# ------------------------------------------------------------ oracle pins (CPU)
def test_oracle_rotation_matches_reference(rot):
    for j in (2, 3, 4):
        b = f"rot16_j{j}"
        th = float(rot[b + "_theta"])
        L = rot[b + "_w"].shape[1]
        assert orc.rel_err(orc.rotate_to_north(rot[b + "_w"], th), rot[b + "_dense"]) <= 1e-14
        assert orc.rel_err(orc.rotate_from_north(rot[b + "_dense"], L, th), rot[b + "_back"]) <= 1e-14
    assert orc.rel_err(orc.rotate_from_north(rot["rot8_dense_in"], 8, float(rot["rot8_theta"])),
                       rot["rot8_from"]) <= 1e-14
    assert orc.rel_err(orc.rotate_to_north(rot["rot_pi_w"], float(rot["rot_pi_theta"])), rot["rot_pi_dense"]) == 0.0
    d = orc.rotate_to_north(rot["rot48_w"], float(rot["rot48_theta"]))
    assert orc.rel_err(d[rot["rot48_idx"]], rot["rot48_val"]) <= 1e-14
    assert orc.rel_err(orc.rotate_from_north(d, 48, float(rot["rot48_theta"])), rot["rot48_back"]) <= 1e-14


def test_oracle_edge_columns_match_reference(rot):
    th = float(rot["rot48_theta"])
    for ell in (0, 1, 17, 47):
        pos, neg = orc.edge_columns(ell, th)
        np.testing.assert_allclose(np.stack([pos, neg]), rot[f"edge48_{ell}"], rtol=0, atol=1e-14)


def test_plane_offsets():
    from paper_1511_05578_b200.so3 import plane_offset
    assert [plane_offset(l) for l in range(5)] == [0, 1, 10, 35, 84]
    assert plane_offset(1024) == sum((2 * l + 1) ** 2 for l in range(1024))


# ------------------------------------------------------------------ GPU parity
gpu = pytest.mark.gpu


def _sc():
    import paper_1511_05578_b200 as sc
    return sc


def host(t):
    return t.detach().cpu().numpy()


@gpu
def test_edge_columns_device(rot):
    sc = _sc()
    th = float(rot["rot48_theta"])
    for ell in (0, 1, 17, 47):
        pos, neg = sc.wigner_d_edge_columns(ell, th)
        np.testing.assert_allclose(np.stack([host(pos), host(neg)]), rot[f"edge48_{ell}"], rtol=0, atol=2e-14)
    # high degrees: the oracle's float64 gammaln closed form vs the device table
    # (extended-precision half log binomials), relative to the column maximum
    for ell in (255, 1023):
        for th in (0.5 * math.pi, 2.2, math.pi):
            pos, neg = sc.wigner_d_edge_columns(ell, th)
            p0, n0 = orc.edge_columns(ell, th)
            assert orc.rel_err(host(pos), p0) <= 1e-11
            assert orc.rel_err(host(neg), n0) <= 1e-11


@gpu
def test_rotation_matches_reference_fixtures(rot):
    sc = _sc()
    for j in (2, 3, 4):
        b = f"rot16_j{j}"
        t = _t(rot[b + "_theta"])
        w = sc.CurveletWignerCoeffs(rot[b + "_w"].shape[1], rot[b + "_w"])
        dense = sc.rotate_to_north(w, 0, t)
        assert orc.rel_err(host(dense.values), rot[b + "_dense"]) <= 1e-13
        back = sc.rotate_from_north(dense, 0, t)
        assert orc.rel_err(host(back.values), rot[b + "_back"]) <= 1e-13
    d = sc.WignerCoeffs(8, values=rot["rot8_dense_in"])
    assert orc.rel_err(host(sc.rotate_from_north(d, 0, _t(rot["rot8_theta"])).values), rot["rot8_from"]) <= 1e-13
    w = sc.CurveletWignerCoeffs(4, rot["rot_pi_w"])
    assert orc.rel_err(host(sc.rotate_to_north(w, 0, _t(rot["rot_pi_theta"])).values), rot["rot_pi_dense"]) <= 1e-13
    t = _t(rot["rot48_theta"])
    w = sc.CurveletWignerCoeffs(48, rot["rot48_w"])
    dense = host(sc.rotate_to_north(w, 0, t).values)
    assert orc.rel_err(dense[rot["rot48_idx"]], rot["rot48_val"]) <= 1e-13
    assert abs(np.sqrt((np.abs(dense) ** 2).sum()) / float(rot["rot48_l2"]) - 1) <= 1e-13
    back = sc.rotate_from_north(sc.WignerCoeffs(48, values=dense), 0, t)
    assert orc.rel_err(host(back.values), rot["rot48_back"]) <= 1e-13


@gpu
@pytest.mark.parametrize("L,spin", [(8, 0), (16, 1), (64, 2)])
def test_round_trip_and_energy(L, spin):
    """The reference's TestFrameRotations.test_round_trip_and_energy on the
    device path (analysis -> so3_forward_curvelet -> rotations)."""
    sc = _sc()
    t = sc.build_tiling(sc.TilingParams(L, spin, 2.0, 1))
    flm = orc.gaussian_flm(L, spin, seed=5, real=False)
    f = sc.SphereSignal(sc.SphereGrid(L), spin, orc.sht_inverse(flm, L, spin))
    c = sc.analyze(f, t)
    for j in range(1, t.params.j_max + 1):
        w = sc.so3_forward_curvelet(c.scale(j))
        dense = sc.rotate_to_north(w, j, t)
        back = sc.rotate_from_north(dense, j, t)
        scale = float(w.values.abs().max())
        assert float((back.values - w.values).abs().max()) <= 1e-12 * max(scale, 1.0)
        wv, cc = host(w.values), w.band_limit - 1
        for ell in range(w.band_limit):
            per_m_dense = (np.abs(host(dense.plane(ell))) ** 2).sum(axis=1)
            per_m_sparse = (np.abs(wv[:, ell, cc - ell: cc + ell + 1]) ** 2).sum(axis=0)
            assert np.abs(per_m_dense - per_m_sparse).max() <= 1e-12 * max(scale, 1.0) ** 2
        # and against the oracle on the same coefficients
        th = float(t.angles[j - t.params.j_min])
        assert orc.rel_err(host(dense.values), orc.rotate_to_north(wv, th)) <= 1e-12


@gpu
def test_identity_rotation_scale(rng):
    sc = _sc()
    t = sc.build_tiling(sc.TilingParams(16, 2, 2.0, 0))
    assert float(t.angles[0]) == pytest.approx(math.pi)
    w = sc.CurveletWignerCoeffs(4, rng.uniform(-1, 1, (2, 4, 7)) + 1j * rng.uniform(-1, 1, (2, 4, 7)))
    # the reference's random() leaves |m| > l empty
    v = host(w.values)
    for ell in range(4):
        v[:, ell, : 3 - ell] = 0
        v[:, ell, 3 + ell + 1:] = 0
    v[1, 0] = 0
    w = sc.CurveletWignerCoeffs(4, v)
    back = sc.rotate_from_north(sc.rotate_to_north(w, 0, t), 0, t)
    assert np.abs(host(back.values) - v).max() <= 1e-13


@gpu
def test_projection_idempotence(rng):
    sc = _sc()
    t = sc.build_tiling(sc.TilingParams(8, 0, 2.0, 0))
    dense = sc.WignerCoeffs.random(8, rng)
    once = sc.rotate_from_north(dense, 2, t)
    again = sc.rotate_from_north(sc.rotate_to_north(once, 2, t), 2, t)
    assert float((again.values - once.values).abs().max()) <= 1e-12


@gpu
def test_errors():
    sc = _sc()
    t = sc.build_tiling(sc.TilingParams(8, 0, 2.0, 1))
    w = sc.CurveletWignerCoeffs.zeros(4)
    with pytest.raises(TypeError):
        sc.rotate_to_north(sc.WignerCoeffs.zeros(4), 1, t)
    with pytest.raises(TypeError):
        sc.rotate_from_north(w, 1, t)
    with pytest.raises(ValueError):
        sc.rotate_to_north(w, 0, t)
    with pytest.raises(ValueError):
        sc.rotate_from_north(sc.WignerCoeffs.zeros(4), t.params.j_max + 1, t)


@gpu
def test_full_size_L1024_properties():
    """C4 finest scale (L_j=1024): the 22.9 GB dense frame.  Round trip
    rotate_from_north(rotate_to_north(w)) = w on the image (w from the
    reference's random() recipe, projected once), per-m energy, and sampled
    planes against the oracle."""
    import torch
    sc = _sc()
    L = 1024
    t = sc.build_tiling(sc.TilingParams(L, 0, 2.0, 3))
    j = t.params.j_max
    th = float(t.angles[j - t.params.j_min])
    g = torch.Generator(device="cuda").manual_seed(0)
    v = torch.complex(torch.rand((2, L, 2 * L - 1), generator=g, device="cuda", dtype=torch.float64) * 2 - 1,
                      torch.rand((2, L, 2 * L - 1), generator=g, device="cuda", dtype=torch.float64) * 2 - 1)
    ell = torch.arange(L, device="cuda")[:, None]
    m = torch.arange(2 * L - 1, device="cuda")[None, :] - (L - 1)
    v *= (m.abs() <= ell)[None]
    v[1, 0] = 0
    w0 = sc.CurveletWignerCoeffs(L, v)
    # project onto the image first: w = P w0 (exact round trip holds on the image)
    w = sc.rotate_from_north(sc.rotate_to_north(w0, j, t), j, t)
    del w0, v
    dense = sc.rotate_to_north(w, j, t)
    back = sc.rotate_from_north(dense, j, t)
    scale = float(w.values.abs().max())
    assert float((back.values - w.values).abs().max()) <= 1e-11 * scale
    wv = host(w.values)
    for ell_ in (0, 1, 100, 511, 1023):
        plane = host(dense.plane(ell_))
        pos, neg = orc.edge_columns(ell_, th)
        c = L - 1
        ref = np.outer(wv[0, ell_, c - ell_: c + ell_ + 1], pos)
        if ell_ > 0:
            ref += np.outer(wv[1, ell_, c - ell_: c + ell_ + 1], neg)
        assert orc.rel_err(plane, ref) <= 1e-11
        per_m_dense = (np.abs(plane) ** 2).sum(axis=1)
        per_m_sparse = (np.abs(wv[:, ell_, c - ell_: c + ell_ + 1]) ** 2).sum(axis=0)
        assert np.abs(per_m_dense - per_m_sparse).max() <= 1e-11 * scale ** 2
    del dense, back
    torch.cuda.empty_cache()


# ------------------------------------------- dense O(L^4) synthesis (8(f) row 4)
@gpu
def test_so3_inverse_general_matches_reference(rot):
    sc = _sc()
    d = sc.WignerCoeffs(6, values=rot["gen_in"])
    out = sc.so3_inverse_general(d, sc.SO3Grid(8, 7, 9))
    assert orc.rel_err(host(out.values), rot["gen_out"]) <= 1e-12
    with pytest.raises(TypeError):
        sc.so3_inverse_general(sc.CurveletWignerCoeffs.zeros(4), sc.SO3Grid(4, 4, 4))
    with pytest.raises(ValueError):
        sc.so3_inverse_general(d, sc.SO3Grid(5, 8, 8))


@gpu
def test_dense_synthesis_matches_sparse_path(rng):
    """The dense transform of the densified outer columns is the
    curvelet-sparse synthesis (the reference's own cross-check)."""
    sc = _sc()
    L = 16
    v = rng.uniform(-1, 1, (2, L, 2 * L - 1)) + 1j * rng.uniform(-1, 1, (2, L, 2 * L - 1))
    for ell in range(L):
        v[:, ell, : L - 1 - ell] = 0
        v[:, ell, L + ell:] = 0
    v[1, 0] = 0
    w = sc.CurveletWignerCoeffs(L, v)
    grid = sc.SO3Grid(L, L, L)
    a = sc.so3_inverse_general(w.densify(), grid)
    b = sc.so3_inverse_curvelet(w, grid)
    assert orc.rel_err(host(a.values), host(b.values)) <= 1e-12


@gpu
def test_north_validation_matches_reference(rot):
    sc = _sc()
    from conftest import reference_tiling
    t = reference_tiling(8, 0, 2.0, 0, 1)  # the generator's second (8, 0, 2, 0) build
    f = sc.SphereSignal(sc.SphereGrid(8), 0, rot["north_map"])
    out = sc.analyze_north_validation(f, t, 2)
    assert orc.rel_err(host(out.values), rot["north_out"]) <= 1e-10
    z = sc.analyze_north_validation(sc.SphereSignal(sc.SphereGrid(8), 0, np.zeros((8, 15), complex)), t, 2)
    assert float(z.values.abs().max()) == 0.0
    with pytest.raises(ValueError):
        sc.analyze_north_validation(f, t, 2, max_band_limit=4)


@gpu
def test_so3_forward_general_matches_reference(rot, rng):
    sc = _sc()
    g = sc.SO3Grid(8, 7, 9)
    out = sc.so3_forward_general(sc.SO3Signal(g, rot["genf_in"]), 6)
    assert orc.rel_err(host(out.values), rot["genf_out"]) <= 1e-12
    # exact on band-limited signals: forward(inverse(w)) = w
    d = sc.WignerCoeffs(6, values=rot["gen_in"])
    back = sc.so3_forward_general(sc.so3_inverse_general(d, g), 6)
    assert orc.rel_err(host(back.values), rot["gen_in"]) <= 1e-12
    with pytest.raises(ValueError):
        sc.so3_forward_general(sc.SO3Signal(g, rot["genf_in"]), 8)
