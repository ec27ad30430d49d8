"""The sharded driver with the CUDA backend at world size 2 (GPU test).

Only one GPU is available per call, and NCCL refuses two ranks on one device,
so both ranks run on cuda:0 with gloo carrying the two collectives (the
broadcast of f_lm on the device tensors; the reduce of the per-scale terms
through a host copy, test-only shim).  What is exercised for real: ScalePlan's
beta-slab split of the scales with 128 <= L_j, CudaBackend (slab analysis and
slab synthesis kernels), the per-rank restricted quadrature tables
(scv_betaq_restrict) and the deterministic merge -- against the single-process
synthesize(analyze(f)) of the same map (transform.py:139-187).  The ranks'
kernels never wait on one another: the collectives are host-level calls
between whole kernels.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, L, spin, q):
    import paper_1511_05578_b200 as sc
    from oracle import scurve_oracle as orc  # checker-side input only
    from paper_1511_05578_b200 import _cabi
    from paper_1511_05578_b200.dist import analyze_sharded, synthesize_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orig_reduce = dist.reduce

    def reduce_via_host(t, dst, op=dist.ReduceOp.SUM, group=None):
        h = torch.view_as_real(t).cpu()
        orig_reduce(h, dst=dst, op=op, group=group)
        t.copy_(torch.view_as_complex(h))

    dist.reduce = reduce_via_host
    try:
        t = sc.build_tiling(sc.TilingParams(L, spin, 2.0, 2))
        f = None
        if rank == 0:
            f = sc.sht_inverse(sc.HarmonicCoeffs(L, spin, orc.gaussian_flm(L, spin, seed=11, real=False)))
        c = analyze_sharded(f, t)
        slabs = {j: (s.b0, s.nb) for j, s in c.scales.items() if isinstance(s, sc.SO3Slab)}
        g = synthesize_sharded(c, t)
        torch.cuda.synchronize()
        ctx = _cabi.context(0)
        # this rank's quadrature tables hold its slab's rows only: the other rank's rows fail loudly
        restricted = True
        for j, (b0, nb) in slabs.items():
            Lj = c.plan.Ljs[j - c.plan.j_min]
            ob0 = 0 if b0 > 0 else nb
            probe = sc.SO3Slab(sc.SO3Grid(Lj, Lj, Lj), ob0, torch.zeros((2 * Lj - 1, 1, 2 * Lj - 1),
                                                                         dtype=torch.complex128, device="cuda"))
            try:
                sc.so3_forward_curvelet_slab(probe)
                restricted = False
            except ValueError:
                pass
        out = {"rank": rank, "slabs": slabs, "owned": sorted(j for j in c.scales if j not in slabs),
               "restricted": restricted}
        if rank == 0:
            # the same map on one process (tables unrestricted again)
            for j, (b0, nb) in slabs.items():
                ctx.betaq_restrict(c.plan.Ljs[j - c.plan.j_min], 0, 0)
            ref = sc.synthesize(sc.analyze(f, t), t)
            out["err"] = float((g.values - ref.values).abs().max() / ref.values.abs().max())
            out["rt"] = float((g.values - f.values).abs().max() / f.values.abs().max())
        q.put(out)
    finally:
        dist.reduce = orig_reduce
        dist.destroy_process_group()


@pytest.mark.parametrize("L,spin", [(256, 0), (256, 2)])
def test_cuda_backend_world2_on_one_gpu(L, spin):
    world = 2
    # the two ranks share this GPU with the test process: hand its cached blocks back first
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, L, spin, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the scales with L_j >= 128 are split into two beta slabs that tile [0, L_j)
    assert set(res[0]["slabs"]) == set(res[1]["slabs"]) and res[0]["slabs"]
    for j in res[0]["slabs"]:
        (a0, an), (b0, bn) = res[0]["slabs"][j], res[1]["slabs"][j]
        assert a0 == 0 and b0 == an and an > 0 and bn > 0
    # every other scale is owned by exactly one rank
    assert not set(res[0]["owned"]) & set(res[1]["owned"])
    assert res[0]["err"] <= 1e-12, res[0]["err"]
    assert res[0]["rt"] <= 1e-11, res[0]["rt"]
    assert all(r["restricted"] for r in res)


@pytest.mark.parametrize("L,spin,world", [(128, 0, 4), (256, 2, 8)])
def test_virtual_rank_shares_tile_the_analysis_and_add_up(L, spin, world):
    """dist.VirtualRank (one rank's share run alone, the mode tools/rank_share.py times): with the
    CUDA backend the shares of all virtual ranks tile analyze()'s scale signals, and their
    per-scale synthesis terms add up to synthesize(analyze(f))."""
    import paper_1511_05578_b200 as sc
    from oracle import scurve_oracle as orc  # checker-side input only
    from paper_1511_05578_b200 import dist as D

    torch.cuda.set_device(0)
    t = sc.build_tiling(sc.TilingParams(L, spin, 2.0, 3))
    p = t.params
    f = sc.sht_inverse(sc.HarmonicCoeffs(L, spin, orc.gaussian_flm(L, spin, seed=4, real=False)))
    full = sc.analyze(f, t)
    ref = sc.synthesize(full, t)
    be = D.CudaBackend()
    terms = torch.zeros((p.scale_count, L * L), dtype=torch.complex128, device="cuda")
    rows = {j: 0 for j in range(p.j_min, p.j_max + 1)}
    plan = None
    try:
        for r in range(world):
            vr = D.VirtualRank(r, world)
            c = D.analyze_sharded(f, t, group=vr, backend=be)
            plan = c.plan
            assert (c.scaling is not None) == (r == 0)
            for j, s in c.scales.items():
                whole = full.scale(j).values
                if isinstance(s, sc.SO3Slab):
                    assert (s.b0, s.nb) in [(b0, nb) for rr, b0, nb in plan.slabs[j] if rr == r]
                    assert orc.rel_err(s.values.cpu().numpy(), whole[:, s.b0:s.b0 + s.nb, :].cpu().numpy()) <= 1e-12
                    rows[j] += s.nb
                    terms[j - p.j_min] += be.scale_term_slab(s, t, j)
                else:
                    assert torch.equal(s.values, whole)
                    rows[j] += s.values.shape[1]
                    terms[j - p.j_min] += be.scale_term(s, t, j, False)
            if r == 0:
                scaling = c.scaling
            be.lift_table_restrictions(plan)
        assert all(rows[j] == full.scale(j).values.shape[1] for j in rows)
        assert plan.slabs, "this size must exercise the beta-slab split"
        acc = torch.zeros(L * L, dtype=torch.complex128, device="cuda")
        for i in range(p.scale_count):
            acc += terms[i]
        g = be.finish(acc, scaling, t, False)
        assert orc.rel_err(g.values.cpu().numpy(), ref.values.cpu().numpy()) <= 1e-12
    finally:
        if plan is not None:
            be.lift_table_restrictions(plan)
