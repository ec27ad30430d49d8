"""Generate the golden fixtures that pin the oracle (and the CUDA path).

Run in the build container, where the reference package is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the UNMODIFIED reference ``scurve`` (never copied into this
repo), runs it on small seeded inputs and writes ``tests/golden/*.npz``.
Those fixtures travel with the repo; nothing at test/bench time reads
/root/reference.  Inputs use the BASELINE.json Gaussian recipe
(C_l=(l+1)^-2) or the reference's own generators (``random_coeffs``,
``CurveletWignerCoeffs.random``), as named per case.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import scurve  # noqa: E402  (the reference)
from scurve import fourier, wigner  # noqa: E402

from oracle.scurve_oracle import gaussian_flm  # noqa: E402  (input recipe only)


def _real_sym_cw(L, rng):
    """Outer-column coefficients whose synthesis is real (mirrors the
    reference test helper's rule, tests/test_so3.py:15-27)."""
    w = scurve.CurveletWignerCoeffs.zeros(L)
    for ell in range(L):
        row = rng.uniform(-1, 1, 2 * ell + 1) + 1j * rng.uniform(-1, 1, 2 * ell + 1)
        if ell == 0:
            row = row.real.astype(complex)
        w.set_row(ell, row)
        if ell > 0:
            ms = np.arange(-ell, ell + 1)
            signs = np.where((ms + ell) % 2 == 0, 1.0, -1.0)
            w.set_row(-ell, signs * np.conj(row[::-1]))
    return w


def wigner_cases(out):
    tab = scurve.build_halfpi_table(12)
    out["halfpi_L12"] = np.concatenate([p.ravel() for p in tab.planes])
    big = scurve.build_halfpi_table(66)
    for ell in (33, 64, 65):
        out[f"halfpi_plane_{ell}"] = big.plane(ell)
    # exact-rational KATs (wigner.py:100-150) at sampled (l, m', m)
    rng = np.random.default_rng(7)
    kat = []
    for _ in range(40):
        ell = int(rng.integers(0, 33))
        mp = int(rng.integers(-ell, ell + 1))
        m = int(rng.integers(-ell, ell + 1))
        kat.append((ell, mp, m, wigner.wigner_d_sum(ell, mp, m, math.pi / 2)))
    out["halfpi_kat"] = np.array(kat, dtype=np.float64)
    # exact values at higher degree (edge and interior), to judge accuracy
    kat2 = []
    for ell in (64, 65, 127):
        for _ in range(12):
            mp = int(rng.integers(-ell, ell + 1))
            m = int(rng.integers(-ell, ell + 1))
            kat2.append((ell, mp, m, wigner.wigner_d_sum(ell, mp, m, math.pi / 2)))
        kat2.append((ell, ell, 0, wigner.wigner_d_sum(ell, ell, 0, math.pi / 2)))
        kat2.append((ell, ell - 1, 3, wigner.wigner_d_sum(ell, ell - 1, 3, math.pi / 2)))
    out["halfpi_kat_hi"] = np.array(kat2, dtype=np.float64)
    out["weight_kernel_7"] = wigner.weight_kernel(14)
    for L in (1, 2, 3, 8, 16):
        K = 2 * L - 1
        x = rng.standard_normal((K, 3)) + 1j * rng.standard_normal((K, 3))
        out[f"wconv_in_{L}"] = x
        out[f"wconv_out_{L}"] = fourier.weighted_convolve(x, axis=0)


def sht_cases(out):
    rng = np.random.default_rng(0)
    for L, s in ((8, 0), (8, 2), (16, 1), (33, 0)):
        flm = scurve.random_coeffs(L, s, rng)
        f = scurve.sht_inverse(flm)
        back = scurve.sht_forward(f)
        out[f"sht_flm_{L}_{s}"] = flm.values
        out[f"sht_map_{L}_{s}"] = f.values
        out[f"sht_fwd_{L}_{s}"] = back.values
        # forward of an arbitrary (not band-limited-consistent) map
        g = rng.standard_normal((L, 2 * L - 1)) + 1j * rng.standard_normal((L, 2 * L - 1))
        out[f"sht_rawmap_{L}_{s}"] = g
        out[f"sht_rawfwd_{L}_{s}"] = scurve.sht_forward(scurve.SphereSignal(scurve.SphereGrid(L), s, g)).values
    for L in (8, 17):
        flm = scurve.random_coeffs(L, 0, rng, real=True)
        f = scurve.sht_inverse_real(flm)
        out[f"shtr_flm_{L}"] = flm.values
        out[f"shtr_map_{L}"] = f.values
        out[f"shtr_fwd_{L}"] = scurve.sht_forward_real(f).values


def so3_cases(out):
    rng = np.random.default_rng(1)
    for L in (4, 8, 13):
        w = scurve.CurveletWignerCoeffs.random(L, rng)
        f = scurve.so3_inverse_curvelet(w, scurve.SO3Grid(L, L, L))
        out[f"so3_w_{L}"] = w.values
        out[f"so3_inv_{L}"] = f.values
        out[f"so3_fwd_{L}"] = scurve.so3_forward_curvelet(f).values
        # forward of an arbitrary SO(3) signal: pins the full linear map
        raw = rng.standard_normal(f.values.shape) + 1j * rng.standard_normal(f.values.shape)
        out[f"so3_raw_{L}"] = raw
        out[f"so3_rawfwd_{L}"] = scurve.so3_forward_curvelet(
            scurve.SO3Signal(scurve.SO3Grid(L, L, L), raw)).values
    for L in (5, 8):
        w = _real_sym_cw(L, rng)
        f = scurve.so3_inverse_curvelet_real(w, scurve.SO3Grid(L, L, L))
        out[f"so3r_w_{L}"] = w.values
        out[f"so3r_inv_{L}"] = f.values
        out[f"so3r_fwd_{L}"] = scurve.so3_forward_curvelet_real(f).values


def tiling_cases(out):
    for (L, s, lam, j0) in ((64, 0, 2.0, 2), (128, 2, 2.0, 2), (512, 0, 2.0, 2),
                            (1024, 0, 2.0, 3), (16, 0, 3.0, 0), (33, 1, 2.5, 1)):
        t = scurve.build_tiling(scurve.TilingParams(L, s, lam, j0))
        key = f"tiling_{L}_{s}_{lam}_{j0}"
        out[key + "_jmax"] = np.array(t.params.j_max)
        out[key + "_kernels"] = t.kernels
        out[key + "_scaling"] = t.scaling
        out[key + "_angles"] = t.angles
        out[key + "_dirpos"] = t.direction_pos
        out[key + "_dirneg"] = t.direction_neg
        pos, neg = scurve.curvelet_harmonics(t, t.params.j_max)
        out[key + "_psipos_jmax"] = pos
        out[key + "_psineg_jmax"] = neg


def transform_cases(out):
    # small full fixtures: every scale stored
    for (L, s, real) in ((16, 0, False), (16, 2, False), (16, 0, True)):
        t = scurve.build_tiling(scurve.TilingParams(L, s, 2.0, 2))
        flm = gaussian_flm(L, s, seed=0, real=real)
        hc = scurve.HarmonicCoeffs(L, s, flm, real=real)
        f = scurve.sht_inverse_real(hc) if real else scurve.sht_inverse(hc)
        c = scurve.analyze_real(f, t) if real else scurve.analyze(f, t)
        g = scurve.synthesize_real(c, t) if real else scurve.synthesize(c, t)
        key = f"xf_{L}_{s}_{int(real)}"
        out[key + "_map"] = f.values
        out[key + "_scaling"] = c.scaling.values
        for i, sig in enumerate(c.scales):
            out[key + f"_scale{i}"] = sig.values
        out[key + "_recon"] = g.values
    # BASELINE config 1 (L=64, s=0, B=2, J0=2): map-level outputs plus
    # per-scale checksums and sampled entries
    L = 64
    t = scurve.build_tiling(scurve.TilingParams(L, 0, 2.0, 2))
    flm = gaussian_flm(L, 0, seed=0, real=True)
    f = scurve.sht_inverse(scurve.HarmonicCoeffs(L, 0, flm))
    c = scurve.analyze(f, t)
    g = scurve.synthesize(c, t)
    out["c1_map"] = f.values
    out["c1_scaling"] = c.scaling.values
    out["c1_recon"] = g.values
    rng = np.random.default_rng(3)
    for i, sig in enumerate(c.scales):
        v = sig.values
        idx = np.stack([rng.integers(0, d, 64) for d in v.shape], axis=1)
        out[f"c1_scale{i}_idx"] = idx
        out[f"c1_scale{i}_val"] = v[tuple(idx.T)]
        out[f"c1_scale{i}_sum"] = v.sum()
        out[f"c1_scale{i}_l2"] = np.array(np.sqrt((np.abs(v) ** 2).sum()))
    w = scurve.so3_forward_curvelet(c.scales[-1])
    out["c1_wlast"] = w.values


def rotation_cases(out):
    """Frame rotation (transform.py:256-297) on the reference's own random
    generators; SURVEY 8(f) row 1."""
    rng = np.random.default_rng(11)
    # scale j=2 of L=16 spin 1, J0=1 (tests/test_transform.py:198-214 shapes)
    t = scurve.build_tiling(scurve.TilingParams(16, 1, 2.0, 1))
    for j, Lw in ((2, 4), (3, 8), (t.params.j_max, 16)):
        w = scurve.CurveletWignerCoeffs.random(Lw, rng)
        dense = scurve.rotate_to_north(w, j, t)
        back = scurve.rotate_from_north(dense, j, t)
        out[f"rot16_j{j}_theta"] = np.array(float(t.angles[j - t.params.j_min]))
        out[f"rot16_j{j}_w"] = w.values
        out[f"rot16_j{j}_dense"] = np.concatenate([p.ravel() for p in dense.planes])
        out[f"rot16_j{j}_back"] = back.values
    # dense random input (projection), L=8, scale 2 of an L=8 J0=0 tiling
    t8 = scurve.build_tiling(scurve.TilingParams(8, 0, 2.0, 0))
    d = scurve.WignerCoeffs.random(8, rng)
    out["rot8_dense_in"] = np.concatenate([p.ravel() for p in d.planes])
    out["rot8_theta"] = np.array(float(t8.angles[2]))
    out["rot8_from"] = scurve.rotate_from_north(d, 2, t8).values
    # identity-angle scale (theta = pi): L=16 spin 2 J0=0, scale 0
    t0 = scurve.build_tiling(scurve.TilingParams(16, 2, 2.0, 0))
    w = scurve.CurveletWignerCoeffs.random(4, rng)
    out["rot_pi_theta"] = np.array(float(t0.angles[0]))
    out["rot_pi_w"] = w.values
    out["rot_pi_dense"] = np.concatenate([p.ravel() for p in scurve.rotate_to_north(w, 0, t0).planes])
    # a larger band limit, sampled: L=48 at the finest scale of an L=48 J0=2 tiling
    t48 = scurve.build_tiling(scurve.TilingParams(48, 0, 2.0, 2))
    j = t48.params.j_max
    w = scurve.CurveletWignerCoeffs.random(48, rng)
    dense = scurve.rotate_to_north(w, j, t48)
    flat = np.concatenate([p.ravel() for p in dense.planes])
    idx = rng.integers(0, flat.size, 512)
    out["rot48_theta"] = np.array(float(t48.angles[j - t48.params.j_min]))
    out["rot48_w"] = w.values
    out["rot48_idx"] = idx
    out["rot48_val"] = flat[idx]
    out["rot48_l2"] = np.array(np.sqrt((np.abs(flat) ** 2).sum()))
    out["rot48_back"] = scurve.rotate_from_north(dense, j, t48).values
    for ell in (0, 1, 17, 47):
        pos, neg = wigner.wigner_d_edge_columns(ell, float(out["rot48_theta"]))
        out[f"edge48_{ell}"] = np.stack([pos, neg])
    # dense O(L^4) synthesis (so3.py:317-346) on a non-square grid, and the
    # north-frame validation path (transform.py:300-322)
    d = scurve.WignerCoeffs.random(6, rng)
    out["gen_in"] = np.concatenate([p.ravel() for p in d.planes])
    out["gen_out"] = scurve.so3_inverse_general(d, scurve.SO3Grid(8, 7, 9)).values
    tn = scurve.build_tiling(scurve.TilingParams(8, 0, 2.0, 0))
    f = scurve.sht_inverse(scurve.random_coeffs(8, 0, rng))
    out["north_map"] = f.values
    out["north_out"] = scurve.analyze_north_validation(f, tn, 2).values
    # dense forward (so3.py:288-314) of a random signal on the same grid, band limit 6
    g = scurve.SO3Grid(8, 7, 9)
    sig = rng.standard_normal(g.shape) + 1j * rng.standard_normal(g.shape)
    out["genf_in"] = sig
    out["genf_out"] = np.concatenate([p.ravel() for p in scurve.so3_forward_general(scurve.SO3Signal(g, sig), 6).planes])


def main_rotation():
    out = {}
    rotation_cases(out)
    path = os.path.join(HERE, "reference_rotation.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {len(out)} arrays to {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


def main_container():
    """SCRV1 files written by the reference's own writers (container.py:152-206)."""
    rng = np.random.default_rng(21)
    t = scurve.build_tiling(scurve.TilingParams(8, 2, 2.0, 1))
    f = scurve.sht_inverse(scurve.random_coeffs(8, 2, rng))
    scurve.container.write_sphere(os.path.join(HERE, "ref_sphere_L8s2.scrv"), f, extra={"seed": 21})
    c = scurve.analyze(f, t)
    scurve.container.write_coeffs(os.path.join(HERE, "ref_coeffs_L8s2.scrv"), c, extra={"note": "golden"})
    t0 = scurve.build_tiling(scurve.TilingParams(8, 0, 2.0, 1))
    fr = scurve.sht_inverse_real(scurve.random_coeffs(8, 0, rng, real=True)) if hasattr(scurve, "sht_inverse_real") else None
    if fr is not None:
        cr = scurve.analyze_real(fr, t0)
        scurve.container.write_coeffs(os.path.join(HERE, "ref_coeffs_L8real.scrv"), cr)
    print("wrote SCRV1 fixtures")


def main_sparsity():
    """Per-scale sparsity statistics exactly as the reference's `sparsity`
    command computes them (cli.py:268-320): analyze / analyze_real, then
    np.histogram of |c|/max and cli.gini_coefficient.  The scale values are
    stored too, so the device statistics can be checked on identical input."""
    from scurve import cli
    rng = np.random.default_rng(31)
    out = {}
    cases = [("s16c", 16, 0, False, 10), ("s16r", 16, 0, True, 7), ("s24s2", 24, 2, False, 12)]
    for name, L, spin, real, bins in cases:
        t = scurve.build_tiling(scurve.TilingParams(L, spin, 2.0, 1))
        flm = scurve.random_coeffs(L, spin, rng, real=real)
        f = scurve.sht_inverse_real(flm) if real else scurve.sht_inverse(flm)
        c = scurve.analyze_real(f, t) if real else scurve.analyze(f, t)
        out[f"{name}_map"] = f.values
        out[f"{name}_meta"] = np.array([L, spin, int(real), bins, t.params.j_min, t.params.j_max])
        for j in range(t.params.j_min, t.params.j_max + 1):
            v = c.scale(j).values
            mags = np.abs(v).ravel()
            top = float(mags.max())
            counts, _ = np.histogram(mags / top, bins=bins, range=(0.0, 1.0))
            out[f"{name}_j{j}_values"] = v
            out[f"{name}_j{j}_stats"] = np.array([mags.size, top, cli.gini_coefficient(mags)])
            out[f"{name}_j{j}_counts"] = counts
    path = os.path.join(HERE, "reference_sparsity.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {len(out)} arrays to {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


def main():
    out = {}
    wigner_cases(out)
    sht_cases(out)
    so3_cases(out)
    tiling_cases(out)
    transform_cases(out)
    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {len(out)} arrays to {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


if __name__ == "__main__":
    if "rotation" in sys.argv[1:]:
        main_rotation()
    elif "container" in sys.argv[1:]:
        main_container()
    elif "sparsity" in sys.argv[1:]:
        main_sparsity()
    else:
        main()
        main_rotation()
        main_container()
        main_sparsity()
