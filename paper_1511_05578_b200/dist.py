"""Scale-sharded multi-GPU analysis / synthesis (one process per GPU).

The curvelet scales j are independent units: analysis of a
scale is a pure function of the broadcast f_lm and psi_j; synthesis of a
scale contributes an additive term to acc_lm.  This module shards the scales
of ONE map over the ranks of a torch.distributed group:

  analysis   rank `src` computes f_lm (SHT) and broadcasts it (NCCL broadcast
             over NVLink, L^2 * 16 B); every rank runs the SO(3) inverse
             transforms of the scales it owns; the scaling signal lives on src.
  synthesis  every rank computes, for each scale it owns, the term
             T_j[lm] = W_{m,+l} psi_+(l) + W_{m,-l} psi_-(l); the terms are
             gathered on `dst`, which adds them in the reference order
             (coarse -> fine, transform.py:164-178), then the scaling part,
             then runs the inverse SHT.  Gathering per-scale terms (instead of
             an arithmetic all-reduce) keeps the merge deterministic and
             bit-identical to the single-GPU path.

Scales are assigned greedily by cost (the (2L_j-1)^2 L_j sample volume),
largest first to the least-loaded rank.  Scale-only sharding stops scaling at
2 GPUs at L=1024 (the two L_j=1024 scales hold 93% of the volume), so every
scale the beta-slab kernels support (complex path, prime-factor K,
128 <= L_j <= 2048) is instead split into `world` contiguous beta slabs, one
per rank: analysis of a slab needs no communication (the closed-form
generation is per beta row), and the synthesis partials of the slabs of a
scale add up to its term (the beta quadrature is a sum over beta rows), so
the same single reduce merges them.  For split scales the merge adds partial
sums, so it is deterministic for a given world size but not bit-identical to
the single-GPU summation order (agreement ~1e-14 relative).  The per-rank compute goes through a
backend object; the default one is the CUDA path of this package.  (The
CPU tests inject the oracle as backend to exercise the sharding logic on the
gloo backend without a GPU.)

For throughput over many maps the better decomposition is maps-per-rank
(bench.py's default multi-GPU mode): no collective at all.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from .transform import scale_band_limit, scaling_band_limit

__all__ = ["ScalePlan", "ShardedCoeffs", "CudaBackend", "analyze_sharded", "roundtrip_sharded_streamed",
           "synthesize_sharded"]


def cuda_splittable(Lj: int, real: bool) -> bool:
    """Scales the beta-slab kernels support (include/scurve_b200.h)."""
    K = 2 * Lj - 1
    return (not real) and 128 <= Lj <= 2048 and (K & (K + 1)) == 0


@dataclass
class ScalePlan:
    """owner[j - j_min] = rank that holds the whole scale j, or -1 when the
    scale is split into beta slabs: slabs[j] = [(rank, b0, nb), ...]."""

    j_min: int
    owner: list
    cost: list
    slabs: dict = field(default_factory=dict)
    Ljs: list = field(default_factory=list)

    @classmethod
    def build(cls, params, world: int, multires: bool = True, real: bool = False,
              splittable=cuda_splittable) -> "ScalePlan":
        js = list(range(params.j_min, params.j_max + 1))
        Ljs = [scale_band_limit(params, j) if multires else params.band_limit for j in js]
        cost = [(2 * L - 1) ** 2 * L for L in Ljs]
        load = [0] * world
        owner = [0] * len(js)
        slabs = {}
        for i, (j, L) in enumerate(zip(js, Ljs)):
            if world > 1 and splittable is not None and splittable(L, real) and L >= world:
                owner[i] = -1
                cuts = [(L * r) // world for r in range(world + 1)]
                slabs[j] = [(r, cuts[r], cuts[r + 1] - cuts[r]) for r in range(world)]
                for r in range(world):
                    load[r] += cost[i] * (cuts[r + 1] - cuts[r]) / L
        for i in sorted(range(len(js)), key=lambda i: (-cost[i], i)):
            if owner[i] == -1:
                continue
            r = min(range(world), key=lambda q: (load[q], q))
            owner[i] = r
            load[r] += cost[i]
        return cls(params.j_min, owner, cost, slabs, Ljs)

    def owned(self, rank: int) -> list:
        """Whole scales held by `rank`."""
        return [self.j_min + i for i, r in enumerate(self.owner) if r == rank]

    def slabs_of(self, rank: int) -> list:
        """(j, b0, nb) beta slabs held by `rank`."""
        return [(j, b0, nb) for j, parts in sorted(self.slabs.items()) for r, b0, nb in parts if r == rank]

    def load(self, rank: int) -> float:
        """Sample volume (cost units) assigned to `rank`."""
        tot = sum(self.cost[j - self.j_min] for j in self.owned(rank))
        for j, b0, nb in self.slabs_of(rank):
            tot += self.cost[j - self.j_min] * nb / self.Ljs[j - self.j_min]
        return tot


@dataclass
class ShardedCoeffs:
    """Distributed CurveletCoeffs: `scales` holds only this rank's scales
    (an SO3Signal for a whole scale, an SO3Slab for a beta slab of a split one)."""

    params: object
    plan: ScalePlan
    scales: dict = field(default_factory=dict)
    scaling: object = None  # on src only
    multires: bool = True
    real: bool = False


class CudaBackend:
    """Per-rank compute on this package's CUDA path."""

    def __init__(self, device=None):
        self.device = device

    def sht_forward(self, f):
        from .sphere import sht_forward, sht_forward_real
        return (sht_forward_real(f) if f.real else sht_forward(f)).values

    def flm_like(self, L):
        return torch.empty(L * L, dtype=torch.complex128, device=torch.device("cuda", torch.cuda.current_device()))

    def scale_inverse(self, flm_vals, t, j, Lj, real):
        from . import _cabi
        from .sphere import HarmonicCoeffs
        from .transform import _scale_wigner, device_tiling
        from .so3 import SO3Grid, so3_inverse_curvelet, so3_inverse_curvelet_real
        dev = flm_vals.device
        ctx = _cabi.context(dev)
        flm = HarmonicCoeffs(t.params.band_limit, 0 if real else t.params.spin, flm_vals, real=real, trusted=True)
        w = _scale_wigner(ctx, flm, device_tiling(t, dev), j, Lj)
        inv = so3_inverse_curvelet_real if real else so3_inverse_curvelet
        return inv(w, SO3Grid(Lj, Lj, Lj))

    def scale_inverse_slab(self, flm_vals, t, j, Lj, b0, nb):
        from . import _cabi
        from .sphere import HarmonicCoeffs
        from .transform import _scale_wigner, device_tiling
        from .so3 import SO3Grid, so3_inverse_curvelet_slab
        dev = flm_vals.device
        ctx = _cabi.context(dev)
        flm = HarmonicCoeffs(t.params.band_limit, t.params.spin, flm_vals, trusted=True)
        w = _scale_wigner(ctx, flm, device_tiling(t, dev), j, Lj)
        return so3_inverse_curvelet_slab(w, SO3Grid(Lj, Lj, Lj), b0, nb)

    def restrict_tables(self, plan, rank: int):
        """Keep only this rank's beta rows of the quadrature table of every split
        scale (scv_betaq_restrict): 8 L_j^2 nb bytes instead of 8 L_j^3 -- at C5 on 8
        ranks 8.6 GB instead of 68.7 GB for L_j = 2048 -- and 1/world of the table
        build's second GEMM.  The context stays restricted (one process per GPU);
        `lift_table_restrictions` undoes it."""
        from . import _cabi
        ctx = _cabi.context(torch.device("cuda", torch.cuda.current_device()) if self.device is None else self.device)
        for j, b0, nb in plan.slabs_of(rank):
            ctx.betaq_restrict(plan.Ljs[j - plan.j_min], b0, nb)

    def lift_table_restrictions(self, plan):
        from . import _cabi
        ctx = _cabi.context(torch.device("cuda", torch.cuda.current_device()) if self.device is None else self.device)
        for Lj in sorted({plan.Ljs[j - plan.j_min] for j in plan.slabs}):
            ctx.betaq_restrict(Lj, 0, 0)

    def scale_term_slab(self, slab, t, j):
        from . import _cabi
        from .so3 import so3_forward_curvelet_slab
        from .transform import device_tiling
        dev = slab.values.device
        ctx = _cabi.context(dev)
        L = t.params.band_limit
        w = so3_forward_curvelet_slab(slab)
        pos, neg = device_tiling(t, dev).psi[j]
        term = torch.zeros(L * L, dtype=torch.complex128, device=dev)
        ctx.call("accumulate", L, slab.grid.L, _cabi.ptr(w.values), _cabi.ptr(pos), _cabi.ptr(neg), _cabi.ptr(term))
        return term

    def scaling_map(self, flm_vals, t, Ls, real):
        from . import _cabi
        from .sphere import HarmonicCoeffs, sht_inverse, sht_inverse_real
        from .transform import _scaling_coeffs, device_tiling
        dev = flm_vals.device
        ctx = _cabi.context(dev)
        flm = HarmonicCoeffs(t.params.band_limit, 0 if real else t.params.spin, flm_vals, real=real, trusted=True)
        s = _scaling_coeffs(ctx, flm, device_tiling(t, dev), Ls, real)
        return sht_inverse_real(s) if real else sht_inverse(s)

    def scale_term(self, sig, t, j, real):
        from . import _cabi
        from .so3 import so3_forward_curvelet, so3_forward_curvelet_real
        from .transform import device_tiling
        dev = sig.values.device
        ctx = _cabi.context(dev)
        L = t.params.band_limit
        w = so3_forward_curvelet_real(sig) if real else so3_forward_curvelet(sig)
        pos, neg = device_tiling(t, dev).psi[j]
        term = torch.zeros(L * L, dtype=torch.complex128, device=dev)
        ctx.call("accumulate", L, sig.grid.L, _cabi.ptr(w.values), _cabi.ptr(pos), _cabi.ptr(neg), _cabi.ptr(term))
        return term

    def finish(self, acc, scaling_sig, t, real):
        from . import _cabi
        from .sphere import HarmonicCoeffs, sht_forward, sht_forward_real, sht_inverse, sht_inverse_real
        from .transform import device_tiling
        dev = acc.device
        ctx = _cabi.context(dev)
        p = t.params
        L = p.band_limit
        dt = device_tiling(t, dev)
        slm = sht_forward_real(scaling_sig) if real else sht_forward(scaling_sig)
        ctx.call("accumulate_scaling", L, slm.band_limit, _cabi.ptr(slm.values), _cabi.ptr(dt.scaling), _cabi.ptr(acc))
        ctx.call("finish_acc", L, p.spin, 1 if real else 0, _cabi.ptr(acc))
        if real:
            return sht_inverse_real(HarmonicCoeffs(L, 0, acc, real=True, trusted=True))
        return sht_inverse(HarmonicCoeffs(L, p.spin, acc, trusted=True))


@dataclass(frozen=True)
class VirtualRank:
    """Stands in for a process group: run rank `rank`'s share of a world-`world`
    decomposition alone, with the collectives skipped (the broadcast input is
    whatever `f` gives, the reduce leaves this rank's terms).  It measures one
    rank's critical path when fewer GPUs than ranks are available
    (tools/rank_share.py); the result is that rank's PARTIAL map, not the map."""

    rank: int
    world: int

    def __post_init__(self):
        if not 0 <= self.rank < self.world:
            raise ValueError(f"rank {self.rank} outside world {self.world}")


def _rank_world(group):
    if isinstance(group, VirtualRank):
        return group.rank, group.world
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _collective(group, world) -> bool:
    return world > 1 and not isinstance(group, VirtualRank)


def analyze_sharded(f, t, group=None, backend=None, src: int = 0, multires: bool = True,
                    real: bool = False, split: bool = True) -> ShardedCoeffs:
    """Analysis of one map with its scales sharded over the group.

    `f` is only read on `src`.  Mirrors transform.analyze (transform.py:139-152)."""
    backend = backend or CudaBackend()
    rank, world = _rank_world(group)
    p = t.params
    L = p.band_limit
    kw = {} if split else {"splittable": None}
    if split and hasattr(backend, "splittable"):
        kw["splittable"] = backend.splittable
    plan = ScalePlan.build(p, world, multires, real=real, **kw)
    if world > 1 and hasattr(backend, "restrict_tables"):
        backend.restrict_tables(plan, rank)
    if rank == src or isinstance(group, VirtualRank):  # a virtual rank has no broadcast to wait for
        flm = backend.sht_forward(f)
    else:
        flm = backend.flm_like(L)
    if _collective(group, world):
        dist.broadcast(flm, src=src, group=group)
    out = ShardedCoeffs(p, plan, multires=multires, real=real)
    for j in plan.owned(rank):
        Lj = scale_band_limit(p, j) if multires else L
        out.scales[j] = backend.scale_inverse(flm, t, j, Lj, real)
    for j, b0, nb in plan.slabs_of(rank):
        out.scales[j] = backend.scale_inverse_slab(flm, t, j, plan.Ljs[j - p.j_min], b0, nb)
    if rank == src:
        Ls = scaling_band_limit(p) if multires else L
        out.scaling = backend.scaling_map(flm, t, Ls, real)
    return out


def synthesize_sharded(c: ShardedCoeffs, t, group=None, backend=None, dst: int = 0):
    """Synthesis of one map from sharded coefficients; the map is returned
    on `dst` (None elsewhere).  Mirrors transform.synthesize (transform.py:155-187)."""
    backend = backend or CudaBackend()
    rank, world = _rank_world(group)
    if rank == dst and c.scaling is None:
        # analyze_sharded forms the scaling signal on its src rank only
        raise ValueError(f"dst={dst} does not hold the scaling signal: synthesize on the analysis src rank")
    p = t.params
    L = p.band_limit
    nsc = p.scale_count
    terms = torch.zeros((nsc, L * L), dtype=torch.complex128,
                        device=next(iter(c.scales.values())).values.device if c.scales else
                        (torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available()
                         and isinstance(backend, CudaBackend) else torch.device("cpu")))
    for j in c.plan.owned(rank):
        terms[j - p.j_min] = backend.scale_term(c.scales[j], t, j, c.real)
    for j, _, _ in c.plan.slabs_of(rank):
        terms[j - p.j_min] = backend.scale_term_slab(c.scales[j], t, j)
    if _collective(group, world):
        # a whole-scale row is nonzero on exactly one rank: sum-reducing the
        # stack moves it without mixing arithmetic (x + 0 == x exactly); the
        # rows of split scales add the slab partials of every rank
        dist.reduce(terms, dst=dst, op=dist.ReduceOp.SUM, group=group)
    if rank != dst:
        return None
    acc = torch.zeros(L * L, dtype=torch.complex128, device=terms.device)
    for i in range(nsc):  # coarse -> fine, the reference order
        acc += terms[i]
    return backend.finish(acc, c.scaling, t, c.real)


def roundtrip_sharded_streamed(f, t, group=None, backend=None, src: int = 0, dst: int = 0, multires: bool = True,
                               slab_rows: int | None = None, consumer=None, split: bool = True):
    """synthesize(analyze(f, t), t) of ONE map over the group, streaming
    beta slabs: no rank ever holds its scale signals whole.

    The scale plan is analyze_sharded's (whole small scales by owner, the
    large scales split into one beta slab per rank); each rank walks its
    slabs in pieces of at most `slab_rows` rows, hands every piece to
    `consumer(j, piece)` and folds it into scale j's synthesis term at once
    (the beta quadrature is a sum over rows), then the (J, L^2) term stack is
    reduced to `dst` as in synthesize_sharded.  Per-rank memory is one piece
    plus the tables, so BASELINE C5 (L=2048, 1.18 TB of coefficients) runs
    with ~147 GB of coefficients per rank never materialised.  Returns the
    reconstructed map on `dst`, None elsewhere.  `f` is read on `src` only.
    """
    backend = backend or CudaBackend()
    rank, world = _rank_world(group)
    p = t.params
    L = p.band_limit
    kw = {} if split else {"splittable": None}
    if split and hasattr(backend, "splittable"):
        kw["splittable"] = backend.splittable
    plan = ScalePlan.build(p, world, multires, real=False, **kw)
    if world > 1 and hasattr(backend, "restrict_tables"):
        backend.restrict_tables(plan, rank)
    flm = backend.sht_forward(f) if rank == src or isinstance(group, VirtualRank) else backend.flm_like(L)
    if _collective(group, world):
        dist.broadcast(flm, src=src, group=group)
    terms = torch.zeros((p.scale_count, L * L), dtype=torch.complex128, device=flm.device)
    for j in plan.owned(rank):
        Lj = scale_band_limit(p, j) if multires else L
        sig = backend.scale_inverse(flm, t, j, Lj, False)
        if consumer is not None:
            consumer(j, sig)
        terms[j - p.j_min] = backend.scale_term(sig, t, j, False)
        del sig
    for j, b0, nb in plan.slabs_of(rank):
        Lj = plan.Ljs[j - p.j_min]
        step = nb if not slab_rows else max(1, min(nb, slab_rows))
        for c0 in range(b0, b0 + nb, step):
            piece = backend.scale_inverse_slab(flm, t, j, Lj, c0, min(step, b0 + nb - c0))
            if consumer is not None:
                consumer(j, piece)
            terms[j - p.j_min] += backend.scale_term_slab(piece, t, j)
            del piece
    scaling = None
    if rank == dst:
        if rank != src:
            raise ValueError("dst must equal src (the scaling signal is formed where f_lm is)")
        Ls = scaling_band_limit(p) if multires else L
        scaling = backend.scaling_map(flm, t, Ls, False)
        if consumer is not None:
            consumer("scaling", scaling)
    if _collective(group, world):
        dist.reduce(terms, dst=dst, op=dist.ReduceOp.SUM, group=group)
    if rank != dst:
        return None
    acc = torch.zeros(L * L, dtype=torch.complex128, device=terms.device)
    for i in range(p.scale_count):  # coarse -> fine, the reference order
        acc += terms[i]
    return backend.finish(acc, scaling, t, False)
