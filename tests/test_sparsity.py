"""Sparsity report (reference cli.py:59-70, 268-320).

reference_sparsity.npz holds, per scale, the reference's analysis values and
the statistics its `sparsity` command computes from them (np.histogram of
|c|/max, cli.gini_coefficient).  CPU: the oracle restatement reproduces them.
GPU: the device kernels (csrc/sparsity.cu) on the same values give the same
integer counts and max, and the Gini to 1e-12; the device pipeline
(analysis + report) matches to the parity tolerance; the streamed report
(beta slabs, no resident coefficients) equals the resident one.
"""

import os

import numpy as np
import pytest

from oracle import scurve_oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sp():
    with np.load(os.path.join(ROOT, "tests", "golden", "reference_sparsity.npz")) as z:
        return {k: z[k] for k in z.files}


def _cases(sp):
    for name in sorted({k.split("_")[0] for k in sp}):
        L, spin, real, bins, j0, j1 = (int(x) for x in sp[f"{name}_meta"])
        yield name, L, spin, bool(real), bins, j0, j1


def test_oracle_matches_reference(sp):
    for name, L, spin, real, bins, j0, j1 in _cases(sp):
        for j in range(j0, j1 + 1):
            n, top, counts, gini = orc.scale_sparsity(sp[f"{name}_j{j}_values"], bins)
            st = sp[f"{name}_j{j}_stats"]
            assert n == int(st[0]) and top == st[1] and gini == st[2]
            assert np.array_equal(counts, sp[f"{name}_j{j}_counts"])


def test_oracle_gini_errors():
    with pytest.raises(ValueError):
        orc.gini_coefficient([])
    with pytest.raises(ValueError):
        orc.gini_coefficient([0.0, 0.0])
    with pytest.raises(ValueError):
        orc.gini_coefficient([-1.0, 2.0])
    assert orc.gini_coefficient([1.0, 1.0, 1.0]) == 0.0


gpu = pytest.mark.gpu


@gpu
def test_device_stats_on_reference_values(sp):
    import torch
    from paper_1511_05578_b200 import sparsity as S
    for name, L, spin, real, bins, j0, j1 in _cases(sp):
        for j in range(j0, j1 + 1):
            v = torch.from_numpy(sp[f"{name}_j{j}_values"]).cuda()
            st = S.scale_statistics(v, bins)
            ref = sp[f"{name}_j{j}_stats"]
            assert st.count == int(ref[0])
            assert abs(st.max_abs - ref[1]) <= 1e-15 * ref[1]
            assert np.array_equal(st.counts, sp[f"{name}_j{j}_counts"]), (name, j)
            assert abs(st.gini - ref[2]) <= 1e-12 * abs(ref[2])


@gpu
def test_device_pipeline_against_reference(sp):
    import paper_1511_05578_b200 as sc
    from paper_1511_05578_b200 import sparsity as S
    from conftest import reference_tiling
    nth = {}
    for name, L, spin, real, bins, j0, j1 in _cases(sp):
        k = nth.get((L, spin, j0), 0)  # the generator's k-th build of these parameters
        nth[(L, spin, j0)] = k + 1
        t = reference_tiling(L, spin, 2.0, j0, k)
        f = sc.SphereSignal(sc.SphereGrid(L), spin, sp[f"{name}_map"], real=real)
        c = sc.analyze_real(f, t) if real else sc.analyze(f, t)
        summary, rows = S.sparsity_report(c, bins)
        assert summary["bins"] == bins and summary["L"] == L and len(rows) == bins * (j1 - j0 + 1)
        for note in summary["scales"]:
            j = note["scale"]
            ref = sp[f"{name}_j{j}_stats"]
            assert note["coefficients"] == int(ref[0])
            assert abs(note["max_abs"] - ref[1]) <= 1e-10 * ref[1]
            assert abs(note["gini"] - ref[2]) <= 1e-10 * abs(ref[2])
            probs = [r[5] for r in rows if r[1] == j]
            ref_p = sp[f"{name}_j{j}_counts"] / ref[0]
            # counts can only move across a bin edge the 1e-14-level value
            # differences straddle: allow one coefficient per bin
            assert np.abs(np.array(probs) - ref_p).max() <= 1.0 / ref[0] + 1e-15


@gpu
def test_gini_random_against_oracle(rng):
    import torch
    from paper_1511_05578_b200 import sparsity as S
    x = rng.standard_normal(3_000_001) ** 2
    g = S.gini_coefficient(torch.from_numpy(x).cuda())
    assert abs(g - orc.gini_coefficient(x)) <= 1e-12
    with pytest.raises(ValueError):
        S.gini_coefficient(torch.zeros(5, dtype=torch.float64))
    with pytest.raises(ValueError):
        S.gini_coefficient(torch.tensor([-1.0, 2.0]))


@gpu
def test_streamed_equals_resident():
    """L=256 (the finest scales are slab-streamed): identical integer counts
    and max, Gini to rounding, with small slabs (several per scale)."""
    import paper_1511_05578_b200 as sc
    from paper_1511_05578_b200 import sparsity as S
    L = 256
    t = sc.build_tiling(sc.TilingParams(L, 0, 2.0, 2))
    fmap = orc.sht_inverse(orc.gaussian_flm(L, 0, seed=3, real=False), L, 0)
    f = sc.SphereSignal(sc.SphereGrid(L), 0, fmap)
    s1, r1 = S.sparsity_report(sc.analyze(f, t), 10)
    s2, r2 = S.sparsity_report_streamed(f, t, 10, slab_bytes=64 << 20)
    for a, b in zip(s1["scales"], s2["scales"]):
        assert a["coefficients"] == b["coefficients"] and a["max_abs"] == b["max_abs"]
        assert abs(a["gini"] - b["gini"]) <= 1e-13
    assert [r[:5] for r in r1] == [r[:5] for r in r2]
    assert [r[5] for r in r1] == [r[5] for r in r2]
