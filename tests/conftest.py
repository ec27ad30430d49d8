import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device")
    config.addinivalue_line("markers", "slow: long-running CPU check")


@pytest.fixture
def rng():
    return np.random.default_rng(0)


@pytest.fixture(scope="session")
def golden():
    path = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def ref_tilings():
    path = os.path.join(ROOT, "tests", "golden", "reference_tilings.npz")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def reference_tiling(L, s, lam, j0, k=0):
    """The k-th tiling with these parameters that the reference's fixture
    generators built (tests/golden/make_golden_tilings.py), as this
    package's Tiling.  Tests comparing transform outputs with reference
    fixtures run on these exact arrays; tests/test_tiling.py pins our own
    build_tiling to them."""
    from paper_1511_05578_b200 import tiling as T
    path = os.path.join(ROOT, "tests", "golden", "reference_tilings.npz")
    key = "t_%d_%d_%s_%d_%d" % (L, s, repr(float(lam)), j0, k)
    with np.load(path) as z:
        a = {n: z[key + "_" + n] for n in ("kernels", "scaling", "dirpos", "dirneg", "angles", "jmax")}
    p = T.TilingParams(L, s, lam, j0, int(a["jmax"]))
    for v in a.values():
        v.setflags(write=False)
    return T.Tiling(p, a["kernels"], a["scaling"], a["dirpos"], a["dirneg"], a["angles"])


@pytest.fixture(autouse=True)
def _gpu_memory_guard(request):
    """GPU tests share one library context per device whose workspace and
    per-L tables grow to the largest size seen (79 GB of quadrature tables
    after the L=2048 cases).  Before each GPU test, if less than 120 GB is
    free, release the torch cache and the context's rebuildable buffers so
    the full-size cases (147 GB of coefficients at L=1024) fit."""
    if request.node.get_closest_marker("gpu") is None:
        yield
        return
    import torch
    if torch.cuda.is_available():
        torch.cuda.empty_cache()
        free, _ = torch.cuda.mem_get_info()
        if free < 150e9:
            from paper_1511_05578_b200 import _cabi
            try:
                _cabi.context(torch.cuda.current_device()).trim()
            except ValueError:
                pass  # pinned by a live graph: nothing to release
    yield
