"""Record the reference's tiling arrays behind every golden fixture.

Run in the build container (the reference is importable there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_tilings.py

The fixture generators (make_golden.py) build their tilings with the
reference's ``build_tiling``, whose Simpson step table is accurate to its
tol = 1e-12 in k_lambda and depends on the process's earlier queries at that
level; sqrt(k_outer - k_inner) amplifies this to ~1e-6 absolute in kappa_j
next to the band edges.  This package's tiling (paper_1511_05578_b200/
tiling.py) integrates k_lambda independently to rounding, so transforms
built from it differ from the reference's fixtures by that amount.  Tests
that compare transform OUTPUTS with reference fixtures therefore run our
transforms on the very tiling arrays the reference used -- recorded here by
re-running the (deterministic) generators with build_tiling wrapped -- while
tests/test_tiling.py pins our own tiling to the reference's at the level of
k_lambda (the squared profiles).

Writes tests/golden/reference_tilings.npz: for the k-th build (k = 0, 1, ...)
of parameters (L, s, lam, j0) in the generators' order, arrays
  t_{L}_{s}_{lam}_{j0}_{k}_{kernels|scaling|dirpos|dirneg|angles|jmax}.
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg  # noqa: E402  (imports the unmodified reference as `scurve`)

scurve = mg.scurve
_orig = scurve.build_tiling
_seen: dict = {}
_out: dict = {}


def _recording_build(params, *a, **kw):
    t = _orig(params, *a, **kw)
    p = t.params
    base = (p.band_limit, p.spin, float(p.lam), p.j_min)
    k = _seen.get(base, 0)
    _seen[base] = k + 1
    key = "t_%d_%d_%s_%d_%d" % (base[0], base[1], repr(base[2]), base[3], k)
    _out[key + "_kernels"] = np.array(t.kernels)
    _out[key + "_scaling"] = np.array(t.scaling)
    _out[key + "_dirpos"] = np.array(t.direction_pos)
    _out[key + "_dirneg"] = np.array(t.direction_neg)
    _out[key + "_angles"] = np.array(t.angles)
    _out[key + "_jmax"] = np.array(p.j_max)
    return t


def main():
    scurve.build_tiling = _recording_build
    # the generators' own fixtures are not rewritten: they write into a
    # temporary directory instead of tests/golden
    tmp = tempfile.mkdtemp()
    mg.HERE = tmp
    try:
        # each generator ran in a fresh process (empty step tables)
        for gen in (mg.main, mg.main_rotation, mg.main_container, mg.main_sparsity):
            scurve.tiling._step_tables.clear()
            gen()
        # the regenerated fixtures must equal the committed ones (same generator,
        # same seeds): the recorded tilings are then exactly the ones used
        for name in ("reference_golden.npz", "reference_rotation.npz", "reference_sparsity.npz"):
            with np.load(os.path.join(tmp, name)) as a, np.load(os.path.join(HERE, name)) as b:
                assert sorted(a.files) == sorted(b.files), name
                for k in a.files:
                    assert np.array_equal(a[k], b[k]), (name, k)
    finally:
        scurve.build_tiling = _orig
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_tilings.npz")
    np.savez_compressed(path, **_out)
    print(f"wrote {len(_out)} arrays ({len(_out) // 6} tilings) to {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
