"""Host-side checks of the B200 formulations (no GPU needed).

The CUDA kernels restructure the reference arithmetic (closed-form edge
columns for the analysis, packed Bluestein + even/odd weight split for the
beta stage, symmetry-reduced Delta wedge).  These numpy models of exactly
those formulations are checked against the oracle so a math slip is caught
on the CPU before any GPU time is spent.
"""

import math

import numpy as np
import pytest
from scipy.special import gammaln

from oracle import scurve_oracle as orc
from paper_1511_05578_b200.wigner import wedge_index, wedge_plane


def test_wedge_symmetries_reconstruct_planes():
    L = 14
    planes = orc.halfpi_planes(L)
    wedge = np.zeros(L * (L + 1) * (L + 2) // 6)
    for l in range(L):
        for a in range(l + 1):
            for b in range(a + 1):
                k, s = wedge_index(l, a, b)
                assert s == 1.0
                wedge[k] = planes[l][a + l, b + l]
    for l in range(L):
        np.testing.assert_allclose(wedge_plane(wedge, l), planes[l], rtol=0, atol=1e-15)


def _edge_d(l, m, n_sign, beta):
    """closed-form d^l_{m, +-l}(beta) as in csrc/so3.cu."""
    hlb = 0.5 * (gammaln(2 * l + 1) - gammaln(l + m + 1) - gammaln(l - m + 1))
    ls, lc = math.log(math.sin(beta / 2)), math.log(math.cos(beta / 2))
    if n_sign >= 0:
        return math.exp(hlb + (l - m) * ls + (l + m) * lc)
    sgn = -1.0 if (l - m) % 2 else 1.0
    return sgn * math.exp(hlb + (l + m) * ls + (l - m) * lc)


def model_so3_inverse(w):
    L = w.shape[1]
    K = 2 * L - 1
    c = L - 1
    betas = math.pi * (2 * np.arange(L) + 1) / K
    T = np.zeros((K, L, K), complex)
    for n in range(-(L - 1), L):
        l = abs(n)
        fac = (2 * l + 1) / (8 * math.pi ** 2)
        for b in range(L):
            for m in range(-l, l + 1):
                T[n % K, b, m % K] = fac * w[0 if n >= 0 else 1, l, c + m] * _edge_d(l, m, n, betas[b])
    T = np.fft.ifft(T, axis=2) * K
    return np.fft.ifft(T, axis=0) * K


@pytest.mark.parametrize("L", [2, 4, 8, 13])
def test_closed_form_analysis(L):
    rng = np.random.default_rng(L)
    w = np.zeros((2, L, 2 * L - 1), complex)
    c = L - 1
    for l in range(L):
        for sh in range(2 if l else 1):
            w[sh, l, c - l:c + l + 1] = rng.uniform(-1, 1, 2 * l + 1) + 1j * rng.uniform(-1, 1, 2 * l + 1)
    ref = orc.so3_inverse_curvelet(w)
    assert orc.rel_err(model_so3_inverse(w), ref) <= 1e-13


def _beta_tables(L):
    K = 2 * L - 1
    P = max(16, 1 << math.ceil(math.log2(4 * L - 3)))
    b = np.arange(K)
    A = np.exp(-1j * math.pi * ((b * b) % (2 * K)) / K)
    h = np.zeros(P, complex)
    for j in range(-(3 * L - 3), L):
        h[j % P] = np.exp(1j * math.pi * ((j * j) % (2 * K)) / K)
    mpp = np.arange(-(L - 1), L)
    C = np.exp(-1j * math.pi * ((mpp * mpp + mpp) % (2 * K)) / K) / K
    def we(k):
        k = np.asarray(k)
        with np.errstate(divide="ignore"):
            return np.where(k % 2 == 0, 2.0 / (1.0 - k.astype(float) ** 2), 0.0)
    v = np.zeros(P, complex)
    q = np.arange(4 * L - 3)
    v[q] = we(2 * (L - 1) - q)
    Aalt = np.array([np.sum(we(mpp - mp) * np.where(mpp % 2, -1.0, 1.0)) for mp in mpp])
    return dict(K=K, P=P, A=A, Hf=np.fft.fft(h) / P, C=C, Vf=np.fft.fft(v) / P, Aalt=Aalt)


def model_beta_pair(sE, sO, T, L):
    """Packed pair: returns (Y_E, Y_O) over m' in [-(L-1), L-1] (no pref)."""
    K, P = T["K"], T["P"]
    def ext(s, p):
        e = np.empty(K, complex)
        e[:L] = s
        e[L:] = p * s[L - 2::-1]
        return e
    u = np.zeros(P, complex)
    u[:K] = (ext(sE, 1) + ext(sO, -1)) * T["A"]
    cc = np.fft.ifft(np.fft.fft(u) * T["Hf"]) * P
    mpp = np.arange(-(L - 1), L)
    F = T["C"] * cc[mpp % P]
    g = 2.0 / K * sO[L - 1]
    alt = np.where(mpp % 2, -1.0, 1.0)
    G = F - 0.5 * g * alt
    z = np.zeros(P, complex)
    z[:K] = G
    E = (np.fft.ifft(np.fft.fft(z) * T["Vf"]) * P)[3 * L - 3 + mpp]
    Fr = F[::-1]
    XE = 0.5 * (F + Fr - g * alt)
    XO = 0.5 * (F - Fr + g * alt)
    def sh(x, d):  # x[k+d] with zeros outside
        y = np.zeros_like(x)
        if d > 0:
            y[:-d] = x[d:]
        else:
            y[-d:] = x[:d]
        return y
    Er = E[::-1]
    YE = 0.5 * (E + Er) + 0.5j * math.pi * (sh(XE, 1) - sh(XE, -1))
    YO = 0.5 * (E - Er) + 0.5 * g * T["Aalt"] + 0.5j * math.pi * (sh(XO, 1) - sh(XO, -1))
    return YE, YO


@pytest.mark.parametrize("L", [1, 2, 3, 5, 8, 17, 33])
def test_packed_beta_stage(L):
    rng = np.random.default_rng(L)
    T = _beta_tables(L)
    sE = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    sO = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    YE, YO = model_beta_pair(sE, sO, T, L)
    refE = orc.beta_to_bins(sE[:, None], L, 1.0, 0, 1.0)[:, 0]
    refO = orc.beta_to_bins(sO[:, None], L, -1.0, 0, 1.0)[:, 0]
    scale = max(np.abs(refE).max(), np.abs(refO).max())
    assert np.abs(YE - refE).max() <= 1e-13 * scale
    assert np.abs(YO - refO).max() <= 1e-13 * scale


# ---------------------------------------------------------------------------
# beta quadrature table (csrc/betaq.cu): the synthesis beta stage + Delta
# contraction of one column (n, m) is a real linear functional of its L beta
# samples, W_mn = sum_b S(b) q_nm(b).  Model of the kernel's real-arithmetic
# formulas, checked against unit-vector probes of the oracle pipeline.
# ---------------------------------------------------------------------------
def model_betaq(L, l, m, planes, pref):
    """q_{n=+l, m}(b), b < L, exactly as k_betaq_build evaluates it."""
    K = 2 * L - 1
    D = planes[l]
    mp = np.arange(-l, l + 1)
    c = D[:, m + l] * D[:, 2 * l]                  # Delta_{m'm} Delta_{m'l}
    cb = np.zeros(2 * L + 2)
    cb[mp + L] = c
    mpp = np.arange(L)
    d = mpp[:, None] - mp[None, :]
    ue = np.where(d % 2 == 0, 2.0 / (1.0 - np.where(d % 2 == 0, d, 0).astype(float) ** 2), 0.0) @ c
    even = (l + m) % 2 == 0
    mn = m - l
    f = pref / K
    b = np.arange(L - 1)
    th = np.pi * np.outer(2 * b + 1, np.arange(1, L)) / K
    q = np.empty(L)
    if even:
        acc = ue[0] + 2.0 * (np.cos(th) @ ue[1:])
        q[:L - 1] = 2.0 * f * (-acc if (mn // 2) % 2 else acc)
    else:
        acc = np.sin(th) @ ue[1:]
        q[:L - 1] = 4.0 * f * (-acc if ((mn - 1) // 2) % 2 else acc)
    full = np.arange(-(L - 1), L)
    sg = np.where(full % 2, -1.0, 1.0)
    u = np.where((full < 0) & (not even), -ue[np.abs(full)], ue[np.abs(full)])
    te = (sg * u).sum()
    to = (sg * (cb[full - 1 + L] - cb[full + 1 + L])).sum()
    if even:
        v = -te if (mn // 2) % 2 else te
    else:
        v = 0.5 * math.pi * (-to if ((mn + 1) // 2) % 2 else to)
    q[L - 1] = f * v
    return q


@pytest.mark.parametrize("L", [2, 3, 6, 9, 16])
def test_beta_quadrature_table(L):
    K = 2 * L - 1
    planes = orc.halfpi_planes(L)
    worst = 0.0
    for n in range(-(L - 1), L):
        l = abs(n)
        probe = np.zeros((L, 2 * l + 1), complex)
        for b in range(L):
            W1 = np.zeros((1, L, K), complex)
            W1[0, b, :] = 1.0
            probe[b] = orc.so3_forward_rows(W1, [n], planes, L)[0]
        assert np.abs(probe.imag).max() <= 1e-13 * max(1.0, np.abs(probe).max())
        for m in range(-l, l + 1):
            if n >= 0:
                q = model_betaq(L, l, m, planes, 4 * math.pi ** 2)
            else:   # q_{-l,m} = (-1)^{l+m} q_{l,-m}
                q = (-1) ** ((l + m) % 2) * model_betaq(L, l, -m, planes, 4 * math.pi ** 2)
            worst = max(worst, np.abs(q - probe[:, m + l].real).max())
    assert worst <= 1e-13
