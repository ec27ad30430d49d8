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


def test_private_graph_survives_eager_growth():
    """A graph captured at a small band limit owns a private context (the
    default), so an eager call at a larger band limit on the same device --
    which grows the shared context's scratch, Delta and cuFFT buffers -- can
    not move memory the graph replays against: the replay stays bit-identical."""
    import paper_1511_05578_b200 as sc
    L = 32
    t = sc.build_tiling(sc.TilingParams(L, 0, 2.0, 2))
    g = sc.GraphedRoundTrip(t)
    fmap = orc.sht_inverse(orc.gaussian_flm(L, 0, seed=3, real=False), L, 0)
    f = sc.SphereSignal(sc.SphereGrid(L), 0, fmap)
    first = g(f.values).values.clone()
    torch.cuda.synchronize()
    Lb = 256
    tb = sc.build_tiling(sc.TilingParams(Lb, 0, 2.0, 2))
    fb = sc.sht_inverse(sc.HarmonicCoeffs(Lb, 0, orc.gaussian_flm(Lb, 0, seed=4, real=False)))
    sc.synthesize(sc.analyze(fb, tb), tb)
    from paper_1511_05578_b200 import _cabi
    _cabi.context(0).trim()  # frees the shared context's scratch outright
    again = g(f.values).values
    torch.cuda.synchronize()
    assert torch.equal(again, first)
    g.close()


def test_shared_context_graph_pins_the_context():
    """With private_context=False the graph replays against the shared
    context's buffers; while it lives, freeing or moving them is refused."""
    import paper_1511_05578_b200 as sc
    from paper_1511_05578_b200 import _cabi
    L = 32
    t = sc.build_tiling(sc.TilingParams(L, 0, 2.0, 2))
    g = sc.GraphedRoundTrip(t, private_context=False)
    ctx = _cabi.context(0)
    with pytest.raises(ValueError, match="pinned"):
        ctx.trim()
    fmap = orc.sht_inverse(orc.gaussian_flm(L, 0, seed=5, real=False), L, 0)
    out = g(fmap).values.clone()
    torch.cuda.synchronize()
    assert orc.rel_err(out.cpu().numpy(), fmap) <= 1e-11
    g.close()
    ctx.trim()  # released: allowed again
