"""Scale-sharded analysis/synthesis over torch.distributed (gloo, world 2, CPU).

The sharding driver (paper_1511_05578_b200/dist.py) is exercised with the
CPU oracle injected as the per-rank compute backend, so the collective
logic (broadcast of f_lm, per-scale ownership, beta-slab splitting of the
large scales, deterministic merge of the per-scale synthesis terms) is
checked without a GPU.  Whole scales must equal the single-process oracle
exactly; slabs are exact slices of it; the merged map, which adds slab
partial sums, agrees to rounding.
"""

import math
import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import scurve_oracle as orc
from paper_1511_05578_b200 import tiling as T
from paper_1511_05578_b200.dist import ScalePlan, analyze_sharded, roundtrip_sharded_streamed, synthesize_sharded


class OracleBackend:
    """CPU restatement standing in for the CUDA path (test only)."""

    def __init__(self, L, spin, split_min=None):
        self.L, self.spin = L, spin
        if split_min is not None:
            self.splittable = lambda Lj, real: (not real) and Lj >= split_min

    def sht_forward(self, f):
        return torch.from_numpy(orc.sht_forward(f, self.L, self.spin))

    def flm_like(self, L):
        return torch.empty(L * L, dtype=torch.complex128)

    def scale_inverse(self, flm, t, j, Lj, real):
        pos, neg = T.curvelet_harmonics(t, j)
        w = orc.scale_wigner(flm.numpy(), pos, neg, Lj)
        vals = orc.so3_inverse_curvelet(w)
        return types.SimpleNamespace(values=torch.from_numpy(vals), grid=types.SimpleNamespace(L=Lj))

    def scale_inverse_slab(self, flm, t, j, Lj, b0, nb):
        full = self.scale_inverse(flm, t, j, Lj, False)
        return types.SimpleNamespace(values=full.values[:, b0:b0 + nb, :].clone(), b0=b0,
                                     grid=types.SimpleNamespace(L=Lj))

    def scale_term_slab(self, slab, t, j):
        # the forward transform is linear in the signal and its beta sum runs
        # over rows: the slab's partial is the transform of the zero-padded slab
        Lj = slab.grid.L
        K = 2 * Lj - 1
        full = torch.zeros((K, Lj, K), dtype=torch.complex128)
        full[:, slab.b0:slab.b0 + slab.values.shape[1], :] = slab.values
        return self.scale_term(types.SimpleNamespace(values=full), t, j, False)

    def scaling_map(self, flm, t, Ls, real):
        return orc.sht_inverse(orc.scaling_coeffs(flm.numpy(), t.scaling, Ls), Ls, 0)

    def scale_term(self, sig, t, j, real):
        w = orc.so3_forward_curvelet(sig.values.numpy())
        pos, neg = T.curvelet_harmonics(t, j)
        L = self.L
        term = np.zeros(L * L, dtype=complex)
        Lj = w.shape[1]
        cc = Lj - 1
        for ell in range(1, Lj):
            if pos[ell] == 0.0 and neg[ell] == 0.0:
                continue
            term[ell * ell:(ell + 1) ** 2] = (w[0, ell, cc - ell:cc + ell + 1] * pos[ell]
                                              + w[1, ell, cc - ell:cc + ell + 1] * neg[ell])
        return torch.from_numpy(term)

    def finish(self, acc, scaling_sig, t, real):
        acc = acc.numpy().copy()
        Ls = scaling_sig.shape[0]
        slm = orc.sht_forward(scaling_sig, Ls, 0)
        for ell in range(Ls):
            a = t.scaling[ell]
            if a == 0.0:
                continue
            a = a * math.sqrt(4.0 * math.pi / (2 * ell + 1))
            acc[ell * ell:(ell + 1) ** 2] += a * slm[ell * ell:(ell + 1) ** 2]
        acc[:self.spin * self.spin] = 0.0
        return orc.sht_inverse(acc, self.L, self.spin)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, L, spin, q, split_min=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = T.build_tiling(T.TilingParams(L, spin, 2.0, 1))
        be = OracleBackend(L, spin, split_min)
        f = orc.sht_inverse(orc.gaussian_flm(L, spin, seed=3, real=False), L, spin)
        c = analyze_sharded(f if rank == 0 else None, t, backend=be)
        g = synthesize_sharded(c, t, backend=be)
        q.put((rank, {j: (getattr(s, "b0", None), s.values.numpy()) for j, s in c.scales.items()},
               None if g is None else np.asarray(g)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("L,spin,split_min", [(16, 0, None), (16, 2, None), (16, 0, 8), (16, 2, 4)])
def test_sharded_matches_single_process(L, spin, split_min):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, L, spin, q, split_min)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    t = T.build_tiling(T.TilingParams(L, spin, 2.0, 1))
    psi = [T.curvelet_harmonics(t, j) for j in range(t.params.j_min, t.params.j_max + 1)]
    f = orc.sht_inverse(orc.gaussian_flm(L, spin, seed=3, real=False), L, spin)
    smap, scales = orc.analyze(f, L, spin, 2.0, 1, t.params.j_max, psi, t.scaling)
    gref = orc.synthesize(smap, scales, L, spin, 2.0, 1, t.params.j_max, psi, t.scaling)
    seen = {}
    for rank, sc, g in res:
        for j, (b0, v) in sc.items():
            ref = scales[j - t.params.j_min]
            if b0 is None:
                np.testing.assert_array_equal(v, ref)
                seen[j] = ref.shape[1]
            else:
                np.testing.assert_array_equal(v, ref[:, b0:b0 + v.shape[1], :])
                seen[j] = seen.get(j, 0) + v.shape[1]
        if rank == 0:
            if split_min is None:
                np.testing.assert_array_equal(g, gref)
            else:
                assert np.abs(g - gref).max() <= 1e-12 * np.abs(gref).max()
        else:
            assert g is None
    # every scale is covered once: whole, or by slabs that partition its beta rows
    assert seen == {j: scales[j - t.params.j_min].shape[1] for j in range(t.params.j_min, t.params.j_max + 1)}


def _worker_streamed(rank, world, port, L, spin, q, split_min):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = T.build_tiling(T.TilingParams(L, spin, 2.0, 1))
        be = OracleBackend(L, spin, split_min)
        f = orc.sht_inverse(orc.gaussian_flm(L, spin, seed=3, real=False), L, spin)
        pieces = []
        g = roundtrip_sharded_streamed(f if rank == 0 else None, t, backend=be, slab_rows=3,
                                       consumer=lambda j, x: pieces.append(
                                           (j, getattr(x, "b0", None), None if isinstance(j, str) else x.values.shape[1])))
        q.put((rank, pieces, None if g is None else np.asarray(g)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("L,spin,split_min", [(16, 2, 4), (16, 0, 8)])
def test_sharded_streamed_round_trip(L, spin, split_min):
    """roundtrip_sharded_streamed (the C5 decomposition): every rank streams its
    beta slabs in 3-row pieces, folds each into its synthesis terms, one
    reduce merges them; the map equals the single-process round trip to
    rounding and every beta row of every scale is visited exactly once."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_streamed, args=(r, world, port, L, spin, q, split_min)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    t = T.build_tiling(T.TilingParams(L, spin, 2.0, 1))
    psi = [T.curvelet_harmonics(t, j) for j in range(t.params.j_min, t.params.j_max + 1)]
    f = orc.sht_inverse(orc.gaussian_flm(L, spin, seed=3, real=False), L, spin)
    smap, scales = orc.analyze(f, L, spin, 2.0, 1, t.params.j_max, psi, t.scaling)
    gref = orc.synthesize(smap, scales, L, spin, 2.0, 1, t.params.j_max, psi, t.scaling)
    rows = {}
    for rank, pieces, g in res:
        for j, b0, nb in pieces:
            if isinstance(j, str):
                assert rank == 0
                continue
            assert nb <= 3 or b0 is None
            rows[j] = rows.get(j, 0) + nb
        if rank == 0:
            assert np.abs(g - gref).max() <= 1e-12 * np.abs(gref).max()
            assert np.abs(g - f).max() <= 1e-11 * np.abs(f).max()
        else:
            assert g is None
    assert rows == {j: scales[j - t.params.j_min].shape[1] for j in range(t.params.j_min, t.params.j_max + 1)}


def test_scale_plan_balances_cost():
    p = T.TilingParams(1024, 0, 2.0, 3)
    for world in (1, 2, 4, 8):
        # scale-only sharding
        plan = ScalePlan.build(p, world, splittable=None)
        owned = [plan.owned(r) for r in range(world)]
        assert sorted(j for o in owned for j in o) == list(range(3, 11))
        if world == 2:  # the two L_j = 1024 scales land on different ranks
            assert plan.owner[-1] != plan.owner[-2]
        # beta-slab splitting of the L_j >= 128 scales: balanced to 1%
        plan = ScalePlan.build(p, world)
        loads = [plan.load(r) for r in range(world)]
        assert max(loads) <= 1.01 * sum(loads) / world
        for j, parts in plan.slabs.items():
            rows = sorted((b0, nb) for _, b0, nb in parts)
            assert rows[0][0] == 0 and sum(nb for _, nb in rows) == plan.Ljs[j - 3]
        # the real path keeps whole scales
        assert not ScalePlan.build(p, world, real=True).slabs


def test_synthesize_sharded_requires_scaling_on_dst():
    """analyze_sharded forms the scaling signal on its src rank only; a dst
    that does not hold it is rejected up front (not after the reduce)."""
    from paper_1511_05578_b200.dist import ShardedCoeffs
    p = T.TilingParams(16, 0, 2.0, 1)
    t = T.build_tiling(p)
    c = ShardedCoeffs(p, ScalePlan.build(p, 1), scaling=None)
    with pytest.raises(ValueError, match="scaling"):
        synthesize_sharded(c, t, backend=OracleBackend(16, 0))


def test_virtual_ranks_cover_the_map_without_a_process_group():
    """VirtualRank runs one rank's share alone (tools/rank_share.py times it on one GPU):
    the shares of all virtual ranks tile the single-process coefficients, and no
    collective is reached (torch.distributed is not initialised here)."""
    from paper_1511_05578_b200.dist import VirtualRank
    L, spin, world = 16, 0, 2
    assert not dist.is_initialized()
    t = T.build_tiling(T.TilingParams(L, spin, 2.0, 1))
    psi = [T.curvelet_harmonics(t, j) for j in range(t.params.j_min, t.params.j_max + 1)]
    f = orc.sht_inverse(orc.gaussian_flm(L, spin, seed=3, real=False), L, spin)
    smap, scales = orc.analyze(f, L, spin, 2.0, 1, t.params.j_max, psi, t.scaling)
    be = OracleBackend(L, spin, 8)
    rows = {j: 0 for j in range(t.params.j_min, t.params.j_max + 1)}
    for r in range(world):
        c = analyze_sharded(f, t, group=VirtualRank(r, world), backend=be)
        assert (c.scaling is not None) == (r == 0)
        assert set(c.scales) == set(c.plan.owned(r)) | {j for j, _, _ in c.plan.slabs_of(r)}
        for j, s in c.scales.items():
            ref = scales[j - t.params.j_min]
            b0 = getattr(s, "b0", None)
            v = s.values.numpy()
            if b0 is None:
                assert np.array_equal(v, ref)
            else:
                assert np.array_equal(v, ref[:, b0:b0 + v.shape[1], :])
            rows[j] += v.shape[1]
        g = synthesize_sharded(c, t, group=VirtualRank(r, world), backend=be)
        assert (g is not None) == (r == 0)
    assert all(rows[j] == scales[j - t.params.j_min].shape[1] for j in rows)
    with pytest.raises(ValueError):
        VirtualRank(2, 2)
