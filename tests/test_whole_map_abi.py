"""scv_analyze / scv_synthesize (one C call per map, transform.py:139-253) against the
per-stage C calls they sequence: bit-identical outputs, same errors."""

import ctypes

import numpy as np
import pytest
import torch

from oracle import scurve_oracle as orc


def test_map_work_bytes_is_exported_and_monotone():
    from paper_1511_05578_b200 import _cabi
    lib = _cabi.load_library()
    a = lib.scv_map_work_bytes(64, 64, 4)
    assert a >= 16 * (64 * 64 + 2 * 64 * 127 + 16)
    assert lib.scv_map_work_bytes(128, 128, 4) > a
    assert lib.scv_map_work_bytes(0, 1, 1) == 0


def _signal(sc, L, spin, real, seed=5):
    flm = orc.gaussian_flm(L, spin, seed=seed, real=real)
    f = sc.sht_inverse(sc.HarmonicCoeffs(L, spin, flm))
    if real:
        f = sc.SphereSignal(f.grid, 0, f.values.real.contiguous(), real=True)
    return f


@pytest.mark.gpu
@pytest.mark.parametrize("L,spin,real,multires,jmin", [(32, 0, False, True, 1), (32, 2, False, True, 2),
                                                       (64, 0, True, True, 2), (24, 1, False, False, 2),
                                                       (128, 0, False, True, 3), (256, 2, False, True, 6)])
def test_whole_map_calls_equal_the_stage_calls(L, spin, real, multires, jmin):
    import paper_1511_05578_b200 as sc
    from paper_1511_05578_b200 import transform as tr
    t = sc.build_tiling(sc.TilingParams(L, spin, 2.0, jmin))
    f = _signal(sc, L, spin, real)
    a = tr._analyze(f, t, multires, real)
    b = tr._analyze_stages(f, t, multires, real)
    assert torch.equal(a.scaling.values, b.scaling.values)
    assert a.scaling.real == b.scaling.real and a.scaling.spin == b.scaling.spin
    assert len(a.scales) == len(b.scales)
    for x, y in zip(a.scales, b.scales):
        assert x.real == y.real and x.grid == y.grid
        assert torch.equal(x.values, y.values)
    g = tr._synthesize(a, t, real)
    h = tr._synthesize_stages(b, t, real)
    assert g.spin == h.spin and g.real == h.real
    assert torch.equal(g.values, h.values)
    assert orc.rel_err(g.values.cpu().numpy(), f.values.cpu().numpy()) <= 1e-11


@pytest.mark.gpu
def test_whole_map_analysis_vs_oracle():
    import paper_1511_05578_b200 as sc
    L, spin, jmin = 32, 2, 2
    p = sc.TilingParams(L, spin, 2.0, jmin)
    t = sc.build_tiling(p)
    flm = orc.gaussian_flm(L, spin, seed=1, real=False)
    fmap = orc.sht_inverse(flm, L, spin)
    c = sc.analyze(sc.SphereSignal(sc.SphereGrid(L), spin, fmap), t)
    psi = [sc.curvelet_harmonics(t, j) for j in range(p.j_min, p.j_max + 1)]
    smap, scales = orc.analyze(fmap, L, spin, 2.0, jmin, p.j_max, psi, t.scaling)
    assert orc.rel_err(c.scaling.values.cpu().numpy(), smap) <= 1e-10
    for x, y in zip(c.scales, scales):
        assert orc.rel_err(x.values.cpu().numpy(), y) <= 1e-10
    g = sc.synthesize(c, t)
    ref = orc.synthesize(smap, scales, L, spin, 2.0, jmin, p.j_max, psi, t.scaling)
    assert orc.rel_err(g.values.cpu().numpy(), ref) <= 1e-10


@pytest.mark.gpu
def test_whole_map_call_rejects_bad_arguments():
    import paper_1511_05578_b200 as sc
    from paper_1511_05578_b200 import _cabi
    from paper_1511_05578_b200 import transform as tr
    L = 16
    t = sc.build_tiling(sc.TilingParams(L, 0, 2.0, 1))
    f = _signal(sc, L, 0, False)
    dev = f.values.device
    ctx = _cabi.context(dev)
    dt = tr.device_tiling(t, dev)
    plan = tr._map_plan(t, dt, True)
    outs = [torch.empty((2 * Lj - 1, Lj, 2 * Lj - 1), dtype=torch.complex128, device=dev) for Lj in plan.Ljs]
    smap = torch.empty((plan.Ls, 2 * plan.Ls - 1), dtype=torch.complex128, device=dev)
    work = torch.empty(plan.work_bytes, dtype=torch.uint8, device=dev)
    sig_arr = plan.sig_arr_t(*[b.data_ptr() for b in outs])

    def call(work_bytes=plan.work_bytes, Ls=plan.Ls, spin=0, real=0):
        ctx.call("analyze", L, spin, real, plan.n, plan.Lj_arr, plan.pos_arr, plan.neg_arr, _cabi.ptr(dt.scaling),
                 Ls, _cabi.ptr(f.values), sig_arr, _cabi.ptr(smap), _cabi.ptr(work), work_bytes)

    call()
    with pytest.raises(ValueError):
        call(work_bytes=plan.work_bytes - 256)
    with pytest.raises(ValueError):
        call(Ls=L + 1)
    with pytest.raises(ValueError):
        call(spin=L)
    with pytest.raises(ValueError):
        call(spin=2, real=1)
    # wrong-dtype scale_out buffers never reach the library
    bad = [torch.empty((2 * Lj - 1, Lj, 2 * Lj - 1), dtype=torch.float64, device=dev) for Lj in plan.Ljs]
    with pytest.raises(TypeError):
        sc.analyze(f, t, scale_out=bad)
    with pytest.raises(ValueError):
        sc.analyze(f, t, scale_out=outs[:-1])
