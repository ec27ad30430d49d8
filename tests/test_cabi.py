"""The C-ABI library loads and exports every symbol include/scurve_b200.h
declares (no compute calls: runs without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_1511_05578_b200 import _cabi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "scurve_b200.h")).read()
    return sorted(set(re.findall(r"\b(scv_[a-z0-9_]+)\s*\(", txt)))


def test_header_and_binding_agree():
    assert set(_declared()) == set(_cabi.EXPORTED)


def test_library_exports_every_symbol():
    if not os.path.exists(_cabi.LIB_PATH):
        pytest.skip("library not built")
    lib = ctypes.CDLL(_cabi.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    lib.scv_version.restype = ctypes.c_int
    assert lib.scv_version() == 102


def test_no_cpu_fallback_without_device(monkeypatch):
    import torch
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _cabi.context(0)
