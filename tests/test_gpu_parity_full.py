"""Oracle parity where the headline is measured (BASELINE C3 / C4) and on the
production synthesis path's full linear map.

* The synthesis beta stage used for every 128 <= L_j <= 2048 (the
  precomputed beta-quadrature table fused into the gamma pass, csrc/betaq.cu)
  against the oracle's so3_forward_curvelet (so3.py:214-244) on
  NON-band-limited inputs: random signals, a probe living only on the last
  beta row (b = L-1, the un-reflected pole node), and thresholded analysis
  coefficients pushed through synthesize (transform.py:155-187).
* C3 (L=512) and C4 (L=1024): every scale of the GPU analysis is compared,
  at sampled gamma frequencies n, with the reference's own route -- the
  Delta-factored bin planes + 2-D inverse FFT of so3.py:247-285
  (oracle.so3_inverse_curvelet(..., n_subset)); the small scales and the
  scaling map in full.  The GPU synthesis is compared, at sampled degrees l,
  with the oracle's beta stage + Delta contraction (so3.py:195-244, oracle
  so3_forward_rows) applied to the single-frequency (gamma, alpha) DFTs of
  the GPU scale signals, summed over scales with the kernels and the scaling
  part as in transform.py:164-187.

Tolerances: <= 1e-10 relative (max|x - ref| / max|ref|) on coefficients and
maps, as in BASELINE.json's north star.
"""

import math

import numpy as np
import pytest
import torch

import paper_1511_05578_b200 as sc
from oracle import scurve_oracle as orc

pytestmark = pytest.mark.gpu

TOL = 1e-10

_PLANES: dict = {}


def host(t):
    return t.detach().cpu().numpy()


def planes_at(ells):
    """Delta planes for the requested degrees (cached across tests)."""
    need = sorted(set(int(e) for e in ells) - set(_PLANES))
    if need:
        _PLANES.update(orc.halfpi_planes_at(max(need) + 1, need))
    return {e: _PLANES[e] for e in ells}


def random_signal(L, seed, real=False):
    rng = np.random.default_rng(seed)
    K = 2 * L - 1
    v = rng.standard_normal((K, L, K))
    if not real:
        v = v + 1j * rng.standard_normal((K, L, K))
    return v


def gamma_slice(F, n):
    """(1/K) sum_g F[g] e^{-i n gamma_g}: the per-n (beta, alpha) plane B_n
    the reference builds before its gamma IFFT (so3.py:281-284), from a
    device signal (K, L, K) (torch; complex result on the host)."""
    K = F.shape[0]
    g = torch.arange(K, device=F.device, dtype=torch.float64)
    ph = torch.exp(-2j * math.pi * n * g / K)
    B = torch.tensordot(ph, F.to(torch.complex128) if not F.is_complex() else F, dims=([0], [0])) / K
    return host(B)


def w1_rows(F, ns):
    """W1[n % K] rows (L, K), alpha in FFT order, of a device signal:
    (1/K^2) sum_{g,a} F e^{-i m alpha_a} e^{-i n gamma_g} (so3.py:198-199),
    the input of the reference's per-n beta stage."""
    K = F.shape[0]
    out = []
    for n in ns:
        B = torch.as_tensor(gamma_slice(F, n), device=F.device)  # (1/K) sum_g
        out.append(host(torch.fft.fft(B, dim=1)) / K)
    return np.stack(out)


def _cw_rows(w, ns):
    return [orc.cw_row(w, n) for n in ns]


# --------------------------------------------- synthesis on non-band-limited input
@pytest.mark.parametrize("L,real", [(128, False), (128, True), (256, False)])
def test_forward_quadrature_path_raw_signal_vs_oracle(L, real):
    """Arbitrary (K, L, K) samples -- not the image of any coefficient set --
    through the production forward transform (beta-quadrature table for
    L_j >= 128) against the oracle's full forward transform."""
    F = random_signal(L, 100 + L, real)
    grid = sc.SO3Grid(L, L, L)
    if real:
        w = sc.so3_forward_curvelet_real(sc.SO3Signal(grid, F, real=True))
        ref = orc.so3_forward_curvelet_real(F)
    else:
        w = sc.so3_forward_curvelet(sc.SO3Signal(grid, F))
        ref = orc.so3_forward_curvelet(F)
    assert orc.rel_err(host(w.values), ref) <= TOL


@pytest.mark.parametrize("L", [128, 256])
def test_forward_quadrature_last_beta_row_probe(L):
    """A signal living only on the last beta node (beta = pi(2L-1)/(2L-1) = pi,
    the node the parity extension does not reflect): exercises the table's
    b = L-1 branch, including the odd weight taps, for every (n, m)."""
    rng = np.random.default_rng(L)
    K = 2 * L - 1
    F = np.zeros((K, L, K), complex)
    F[:, L - 1, :] = rng.standard_normal((K, K)) + 1j * rng.standard_normal((K, K))
    grid = sc.SO3Grid(L, L, L)
    from paper_1511_05578_b200 import _cabi
    ctx = _cabi.context(0)
    w = host(sc.so3_forward_curvelet(sc.SO3Signal(grid, F)).values)
    try:
        ctx.set_option("betaq", 0)  # the per-column FFT beta stage
        w_fft = host(sc.so3_forward_curvelet(sc.SO3Signal(grid, F)).values)
    finally:
        ctx.set_option("betaq", -1)
    ref = orc.so3_forward_curvelet(F)
    assert orc.rel_err(w, ref) <= TOL
    assert orc.rel_err(w_fft, ref) <= TOL


@pytest.mark.parametrize("L,s", [(128, 0), (128, 2)])
def test_synthesize_thresholded_coefficients_vs_oracle(L, s):
    """Hard-thresholded analysis coefficients (the curvelet denoising use of
    synthesize) are not band-limited SO(3) signals: synthesize them on the GPU
    and in the oracle, compare the maps."""
    t = sc.build_tiling(sc.TilingParams(L, s, 2.0, 2))
    p = t.params
    psi = [sc.curvelet_harmonics(t, j) for j in range(p.j_min, p.j_max + 1)]
    flm = orc.gaussian_flm(L, s, seed=7, real=False)
    f = sc.sht_inverse(sc.HarmonicCoeffs(L, s, flm))
    c = sc.analyze(f, t)
    scales = []
    for sig in c.scales:
        v = sig.values
        thr = 0.2 * float(v.abs().max())
        v.mul_((v.abs() >= thr).to(v.dtype))
        scales.append(host(v))
    smap = host(c.scaling.values)
    g = sc.synthesize(c, t)
    ref = orc.synthesize(smap, scales, L, s, 2.0, 2, p.j_max, psi, t.scaling)
    assert orc.rel_err(host(g.values), ref) <= TOL


# ------------------------------------------------- beta slabs at L_j = 512, 1024
@pytest.mark.parametrize("L,b0,nb", [(512, 200, 16), (1024, 1000, 8)])
def test_forward_slab_sampled_n_vs_oracle(L, b0, nb):
    """so3_forward_curvelet_slab of a random beta slab (the multi-GPU shard of
    a large scale) against the oracle's per-n beta stage + Delta contraction
    (so3.py:231-243) on the slab zero-padded to the full beta range."""
    K = 2 * L - 1
    rng = np.random.default_rng(L + b0)
    vals = rng.standard_normal((K, nb, K)) + 1j * rng.standard_normal((K, nb, K))
    grid = sc.SO3Grid(L, L, L)
    dv = torch.as_tensor(vals, device="cuda")
    w = host(sc.so3_forward_curvelet_slab(sc.SO3Slab(grid, b0, dv)).values)
    ns = [0, 1, -1, 17, -200, 311, L // 2, -(L - 1), L - 1]
    pl = planes_at([abs(n) for n in ns])
    W1 = np.zeros((len(ns), L, K), complex)  # the slab zero-padded to all L beta rows
    W1[:, b0:b0 + nb, :] = w1_rows(dv, ns)
    rows = orc.so3_forward_rows(W1, ns, pl, L)
    got = np.concatenate([orc.cw_row(w, n) for n in ns])
    assert orc.rel_err(got, np.concatenate(rows)) <= TOL
    del dv
    torch.cuda.empty_cache()


# ------------------------------------------------------------ C3 and C4, sampled
def _pipeline_vs_oracle(L, s, J0, seed, ells):
    t = sc.build_tiling(sc.TilingParams(L, s, 2.0, J0))
    p = t.params
    flm = orc.gaussian_flm(L, s, seed=seed, real=(s == 0))
    fmap = orc.sht_inverse(flm, L, s) if L <= 512 else None
    f = sc.sht_inverse(sc.HarmonicCoeffs(L, s, flm))
    if fmap is not None:
        assert orc.rel_err(host(f.values), fmap) <= TOL
    c = sc.analyze(f, t)
    # scaling map in full
    Ls = sc.scaling_band_limit(p)
    smap = orc.sht_inverse(orc.scaling_coeffs(flm, t.scaling, Ls), Ls, 0)
    assert orc.rel_err(host(c.scaling.values), smap) <= TOL
    pl = planes_at(ells)
    # analysis, every scale: full for L_j <= 256, sampled gamma frequencies above
    worst = 0.0
    for j, sig in zip(range(p.j_min, p.j_max + 1), c.scales):
        Lj = sig.grid.L
        pos, neg = sc.curvelet_harmonics(t, j)
        w = orc.scale_wigner(flm, pos, neg, Lj)
        if Lj <= 256:
            worst = max(worst, orc.rel_err(host(sig.values), orc.so3_inverse_curvelet(w)))
            continue
        ns = [n for l in ells if l < Lj for n in ((l, -l) if l else (0,))]
        ref = orc.so3_inverse_curvelet(w, pl, n_subset=ns)
        got = np.stack([gamma_slice(sig.values, n) for n in ns])
        worst = max(worst, orc.rel_err(got, ref))
    assert worst <= TOL, worst
    # synthesis at sampled degrees: acc_lm = sum_j W_j(m, +-l) psi_+-(l) + scaling
    g = sc.synthesize(c, t)
    acc = host(sc.sht_forward(g).values)
    slm = orc.sht_forward(smap, Ls, 0)
    ref_rows, got_rows = [], []
    for l in ells:
        if l < abs(s):
            continue
        row = np.zeros(2 * l + 1, complex)
        for j, sig in zip(range(p.j_min, p.j_max + 1), c.scales):
            Lj = sig.grid.L
            if l >= Lj or l == 0:
                continue
            pos, neg = sc.curvelet_harmonics(t, j)
            if pos[l] == 0.0 and neg[l] == 0.0:
                continue
            rws = orc.so3_forward_rows(w1_rows(sig.values, [l, -l]), [l, -l], pl, Lj)
            row += rws[0] * pos[l] + rws[1] * neg[l]
        if l < Ls:
            row += t.scaling[l] * math.sqrt(4.0 * math.pi / (2 * l + 1)) * slm[l * l:(l + 1) ** 2]
        ref_rows.append(row)
        got_rows.append(acc[l * l:(l + 1) ** 2])
    assert orc.rel_err(np.concatenate(got_rows), np.concatenate(ref_rows)) <= TOL
    rt = float((g.values - f.values).abs().max() / f.values.abs().max())
    assert rt <= 1e-11, rt
    del c, g
    torch.cuda.empty_cache()


def test_c3_L512_pipeline_vs_oracle():
    """BASELINE configs[2] (C3): L=512, spin 0, lambda=2, J0=2 (map 0 of the
    batch; maps are independent).  Scales 8..256 and the scaling map in full,
    both L_j=512 scales at 9 gamma frequencies, synthesis at 6 degrees."""
    _pipeline_vs_oracle(512, 0, 2, 0, [0, 3, 130, 255, 300, 511])


def test_c4_L1024_pipeline_vs_oracle():
    """BASELINE configs[3] (C4, the headline): L=1024, spin 0, lambda=2, J0=3.
    Scales 16..256 and the scaling map in full; the L_j=512 scale and both
    L_j=1024 scales at sampled gamma frequencies; synthesis at 6 degrees."""
    _pipeline_vs_oracle(1024, 0, 3, 0, [0, 9, 200, 511, 700, 1023])


@pytest.mark.parametrize("L", [128, 256])
def test_quadrature_table_gemm_build_equals_direct_build(L):
    """The beta-quadrature table (csrc/betaq.cu: the weights that stand for the
    reference's beta FFT, quadrature convolution and Delta contraction,
    so3.py:203-243) built as two tensor-core GEMMs is the table of the direct
    sums: equal to 1e-13 of the table's largest weight."""
    from paper_1511_05578_b200 import _cabi
    ctx = _cabi.context(0)
    n = L ** 3
    tabs = []
    for method in (0, 1):
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        ctx.call("debug_betaq_build", L, method, _cabi.ptr(out), n)
        tabs.append(out)
    torch.cuda.synchronize()
    assert not bool(torch.isnan(tabs[1]).any())
    scale = float(tabs[0].abs().max())
    assert float((tabs[0] - tabs[1]).abs().max()) <= 1e-13 * scale


@pytest.mark.parametrize("L", [256, 512])
def test_quadrature_table_restricted_to_a_beta_slab(L):
    """scv_betaq_restrict (a rank's table in the beta-slab decomposition): the
    slab synthesis with the table cut to the slab's rows is bit-identical to the
    one with the whole table, the table shrinks by L / nb, rows outside fail
    loudly, and lifting the restriction restores the whole transform."""
    from paper_1511_05578_b200 import _cabi
    ctx = _cabi.context(0)
    b0, nb = 96, 64  # L = 512 runs the ring kernels (K = 1023), L = 256 the batched one
    rng = np.random.default_rng(3)
    K = 2 * L - 1
    grid = sc.SO3Grid(L, L, L)
    slab = sc.SO3Slab(grid, b0, torch.as_tensor(rng.standard_normal((K, nb, K)) + 1j * rng.standard_normal((K, nb, K)),
                                                device="cuda"))
    other = sc.SO3Slab(grid, 0, slab.values[:, :8, :].contiguous())
    ctx.betaq_restrict(L, 0, 0)
    ref = sc.so3_forward_curvelet_slab(slab).values.clone()
    ref_other = sc.so3_forward_curvelet_slab(other).values.clone()
    full_bytes = ctx.workspace_bytes()
    try:
        ctx.betaq_restrict(L, b0, nb)
        got = sc.so3_forward_curvelet_slab(slab).values
        assert torch.equal(got, ref)
        assert full_bytes - ctx.workspace_bytes() >= 8 * (L - nb) * L * L * 0.99
        with pytest.raises(ValueError):
            sc.so3_forward_curvelet_slab(other)
        with pytest.raises(ValueError):
            ctx.betaq_restrict(L, L - 3, 8)
    finally:
        ctx.betaq_restrict(L, 0, 0)
    assert torch.equal(sc.so3_forward_curvelet_slab(other).values, ref_other)
