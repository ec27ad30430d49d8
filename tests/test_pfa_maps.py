"""Host-side check of the prime-factor engine's position maps (csrc/pfa.cu).

The K-point DFT engine keeps a row in shared memory as the array
x[n_0]..[n_{D-1}] of the Ruritanian input map and reads the result through
the CRT output map; for K = 2047 the 89 elements of the innermost dimension
are additionally stored in the order the Rader radix-89 stage wants
(pfa.cuh, pfa_stage_rader89).  Every kernel goes through the two 16-bit maps,
so they alone carry the permutations.  This test emulates the stages with
numpy on the maps the library builds (no GPU) and compares with numpy.fft:
replaces part of the reference's scipy.fft calls (so3.py:185-211)."""
import ctypes

import numpy as np
import pytest

from paper_1511_05578_b200 import _cabi

# the plans of csrc/pfa.cuh (composite radices are fine: the factors only have to be coprime)
FACTORS = {15: (3, 5), 63: (7, 9), 255: (3, 5, 17), 511: (7, 73), 1023: (31, 33), 2047: (23, 89),
           4095: (9, 13, 35)}


def _maps(K):
    lib = _cabi.load_library()
    out = (ctypes.c_int * K)()
    inn = (ctypes.c_int * K)()
    assert lib.scv_debug_pfa_maps(K, out, inn) == 0
    return np.array(out), np.array(inn)


def _sigma():
    lib = _cabi.load_library()
    a = (ctypes.c_int * 89)()
    b = (ctypes.c_int * 89)()
    assert lib.scv_debug_r89_sigma(a, b) == 0
    return np.array(a), np.array(b)


@pytest.mark.parametrize("K", sorted(FACTORS))
def test_maps_reproduce_the_dft(K):
    out, inn = _maps(K)
    assert sorted(out) == list(range(K)) and sorted(inn) == list(range(K))
    f = FACTORS[K]
    rng = np.random.default_rng(K)
    x = rng.standard_normal(K) + 1j * rng.standard_normal(K)
    X = np.empty(K, complex)
    X[inn] = x
    A = X.reshape(f)
    sin, sout = _sigma()
    for ax, p in enumerate(f):
        if p == 89 and K == 2047:
            # stage reads element j at sigma_in(j), writes y_k at sigma_out(k)
            A = np.take(A, sin, axis=ax)
            A = np.fft.fft(A, axis=ax)
            B = np.empty_like(A)
            idx = [slice(None)] * A.ndim
            idx[ax] = sout
            B[tuple(idx)] = A
            A = B
        else:
            A = np.fft.fft(A, axis=ax)
    y = A.reshape(K)[out]
    assert np.max(np.abs(y - np.fft.fft(x))) <= 1e-11 * np.max(np.abs(y))


def test_rader_storage_order_is_linear_in_the_lane_coordinates():
    """sigma_in / sigma_out are what the stage's compile-time offsets assume
    (pfa.cuh): pair a = (33 a1 + 12 a2) mod 44 at 1 + 11 a1 + a2 and 44 further,
    outputs at 1 + 2 b2 + (b1 & 1) + 22 (b1 >> 1) and 44 further, the member with
    the + wrap sign first."""
    sin, sout = _sigma()
    assert sorted(sin) == list(range(89)) and sorted(sout) == list(range(89))
    assert sin[0] == 0 and sout[0] == 0
    r = 1
    for a in range(44):
        neg = (a >> 2) & 1
        u, v = (89 - r, r) if neg else (r, 89 - r)
        a1, a2 = a % 4, a % 11
        assert (33 * a1 + 12 * a2) % 44 == a
        assert sin[u] == 1 + 11 * a1 + a2 and sin[v] == 45 + 11 * a1 + a2
        t = 2 * a2 + (a1 & 1) + 22 * (a1 >> 1)
        assert sout[u] == 1 + t and sout[v] == 45 + t
        r = (r * 3) % 89


@pytest.mark.parametrize("K", [1023, 2047])
def test_lane_schedule_is_a_permutation_and_cuts_bank_conflicts(K):
    """The ring kernels' lane schedule (csrc/pfa.cu, pfa_lane_schedule): within every group
    of 32 consecutive elements each element is moved by exactly one lane, to the position
    the plain map gives, and the quarter-warps meet fewer 16-byte bank-group conflicts than
    in natural lane order."""
    lib = _cabi.load_library()
    out = (ctypes.c_int * K)()
    inn = (ctypes.c_int * K)()
    assert lib.scv_debug_pfa_maps(K, out, inn) == 0
    so = (ctypes.c_int * K)()
    si = (ctypes.c_int * K)()
    assert lib.scv_debug_pfa_sched(K, so, si) == 0

    def wavefronts(pos_by_lane):
        w = 0
        for q in range(0, len(pos_by_lane), 8):
            g = [p & 7 for p in pos_by_lane[q:q + 8]]
            w += max(g.count(b) for b in range(8))
        return w

    for plain, sched in ((list(out), list(so)), (list(inn), list(si))):
        nat = got = 0
        for n0 in range(0, K, 32):
            W = min(32, K - n0)
            ent = sched[n0:n0 + W]
            es = sorted(e >> 11 for e in ent)
            assert es == list(range(W))
            for e in ent:
                assert (e & 0x7ff) == plain[n0 + (e >> 11)]
            nat += wavefronts(plain[n0:n0 + W])
            got += wavefronts([e & 0x7ff for e in ent])
        # K = 2047 (the length the schedule was built for): at least 22% fewer wavefronts; the
        # 31 x 33 maps of K = 1023 conflict less in natural order to begin with (r08)
        assert got <= (0.78 if K == 2047 else 0.9) * nat, (got, nat)
