"""CUDA-graph replay of the round trip (GraphedRoundTrip): bit-identical to
the eager analyze + synthesize on the same map, for several maps replayed
through one captured graph, complex and real paths."""

import numpy as np
import pytest
import torch

from oracle import scurve_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("L,spin,real", [(32, 0, False), (64, 2, False), (64, 0, True)])
def test_graph_replay_bit_identical(L, spin, real):
    import paper_1511_05578_b200 as sc
    t = sc.build_tiling(sc.TilingParams(L, spin, 2.0, 2))
    g = sc.GraphedRoundTrip(t, spin=spin, real=real)
    assert g.kernels_per_replay > 0
    for seed in range(3):
        flm = orc.gaussian_flm(L, spin, seed=seed, real=real)
        fmap = orc.sht_inverse(flm, L, spin)
        if real:
            fmap = fmap.real
        f = sc.SphereSignal(sc.SphereGrid(L), spin, fmap, real=real)
        ana, syn = (sc.analyze_real, sc.synthesize_real) if real else (sc.analyze, sc.synthesize)
        c = ana(f, t)
        eager = syn(c, t).values.clone()
        out = g(f.values)
        torch.cuda.synchronize()
        assert torch.equal(out.values, eager)
        for a, b in zip(g.coeffs.scales, c.scales):
            assert torch.equal(a.values, b.values)
        assert orc.rel_err(out.values.cpu().numpy(), fmap) <= 1e-11


@pytest.mark.parametrize("L,spin,real", [(32, 1, False), (64, 0, True)])
def test_batched_lanes_bit_identical(L, spin, real):
    """Seven maps through three concurrent lanes (private contexts, own
    streams): every reconstruction equals the eager round trip of its map."""
    import paper_1511_05578_b200 as sc
    t = sc.build_tiling(sc.TilingParams(L, spin, 2.0, 2))
    b = sc.BatchedRoundTrip(t, lanes=3, spin=spin, real=real)
    maps, eager = [], []
    ana, syn = (sc.analyze_real, sc.synthesize_real) if real else (sc.analyze, sc.synthesize)
    for seed in range(7):
        fmap = orc.sht_inverse(orc.gaussian_flm(L, spin, seed=10 + seed, real=real), L, spin)
        if real:
            fmap = fmap.real
        f = sc.SphereSignal(sc.SphereGrid(L), spin, fmap, real=real)
        maps.append(f.values)
        eager.append(syn(ana(f, t), t).values.clone())
    out = b(torch.stack(maps))
    torch.cuda.synchronize()
    for i in range(7):
        assert torch.equal(out[i], eager[i]), i
    # a second batch through the same lanes (graph-owned buffers reused)
    out2 = b(torch.stack(maps[::-1]))
    torch.cuda.synchronize()
    for i in range(7):
        assert torch.equal(out2[i], eager[6 - i]), i
