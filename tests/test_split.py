"""Two-region pull layout + tiled heavy gather (csrc/gee_split.cu).

The split layout must give the same class stream and the same Z bits as the
one-region layout it is built from (the reducers' sums are exact integers),
and the oracle within tolerance: every tile size (many tiles, one tile, a
partial last tile), both label packings (6-bit for K <= 63, bytes up to 255),
weighted and unit, heavy rows with cold tails, mega rows of several work
items, and runs longer than one warp's piece (SEG_MAX)."""

import numpy as np
import pytest

import oracle
from conftest import rel_err

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2402_04403_b200 import synth  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph, Embedder  # noqa: E402

DEV = torch.device("cuda")


def _graph(scale, s, k, weighted, seed, hub_arcs=0):
    src, dst, w = synth.rmat_edges(scale, s, seed=seed, weighted=weighted)
    if hub_arcs:  # a mega row (several 65 536-arc work items)
        src[:hub_arcs] = 7
    n = 1 << scale
    y = synth.uniform_labels(n, k, seed=seed)
    y[::13] = 0
    return src, dst, w, y, n


@pytest.mark.parametrize("k,weighted,tile", [
    (50, True, 4000), (50, True, None), (5, False, 1235), (100, False, 4096), (255, True, 65536),
])
def test_split_layout_bitwise_equals_one_region(k, weighted, tile):
    src, dst, w, y, n = _graph(17, 1_500_000, k, weighted, seed=k, hub_arcs=150_000)
    g = DeviceGraph.from_edges(src, dst, w, n, device=DEV, pull=True)
    g.prepare_hot(k, enable=True, split=False)
    assert g.n_heavy > 0 and g.n_mega > 0 and g.n_hot > 0
    emb = Embedder(n, k, DEV)
    emb.project(y, g=g)
    z1 = emb.pull(g).clone()
    cls1 = emb.cls[:g.arcs].clone()
    tgt1, off1 = g.targets.clone(), g.offsets.clone()
    assert g.split_heavy(k, tile=tile, keep_unsplit=True)
    assert g.split and g.n_tiles >= 1 and g.n_tails > 0
    if tile and tile < g.n_hot:
        assert g.n_tiles > 1
    # relocation: light rows in place order, heavy rows behind them
    assert int(g.offsets[-1]) == g.light_arcs
    hr = g.heavy_rows.long()
    assert torch.equal(g.offsets[hr + 1] - g.offsets[hr], torch.zeros_like(hr))
    emb2 = Embedder(n, k, DEV)
    emb2.project(y, g=g)
    z2 = emb2.pull(g)
    # the class stream holds the same bytes at the relocated positions
    for r in hr[:50].tolist() + [int(x) for x in torch.randint(0, n, (50,))]:
        a, b = int(off1[r]), int(off1[r + 1])
        if r in set(hr.tolist()):
            i = int((g.heavy_rows.long() == r).nonzero()[0, 0])
            c = int(g.hoff[i])
        else:
            c = int(g.offsets[r])
        assert torch.equal(g.targets[c:c + b - a], tgt1[a:b])
        assert torch.equal(emb2.cls[c:c + b - a], cls1[a:b])
    assert torch.equal(z1.view(torch.int32), z2.view(torch.int32))
    exp = oracle.serial_embed(src.cpu().numpy(), dst.cpu().numpy(), None if w is None else w.cpu().numpy(),
                              y.cpu().numpy(), n, k)
    assert rel_err(z2.cpu().numpy(), exp) <= 1e-4
    # runs: every hot run lies inside one tile, pieces cover the hot runs
    starts, lens = g.seg_start[:g.tail_first], g.seg_len[:g.tail_first].long()
    assert int(lens.max()) <= 2048
    so = g.seg_off.cpu()
    for t in range(g.n_tiles):
        a, b = int(so[t]), int(so[t + 1])
        if a == b:
            continue
        first = g.targets[starts[a:b]].long()
        last = g.targets[starts[a:b] + lens[a:b] - 1].long()
        assert int(first.min()) >= t * g.tile and int(last.max()) < min((t + 1) * g.tile, g.n_hot)
    assert int(g.piece[0]) == 0 and int(g.piece[-1]) == g.tail_first
    assert bool((g.piece[1:] >= g.piece[:-1]).all())
    # every heavy arc is covered exactly once by the runs and tails
    cover = torch.zeros(g.arcs, dtype=torch.int32, device=DEV)
    idx = torch.repeat_interleave(g.seg_start[:g.tail_first + g.n_tails],
                                  g.seg_len[:g.tail_first + g.n_tails].long())
    ramp = torch.arange(idx.numel(), device=DEV) - torch.repeat_interleave(
        torch.cumsum(g.seg_len[:g.tail_first + g.n_tails].long(), 0) - g.seg_len[:g.tail_first + g.n_tails].long(),
        g.seg_len[:g.tail_first + g.n_tails].long())
    cover.index_add_(0, idx + ramp, torch.ones_like(idx, dtype=torch.int32))
    assert int(cover[:g.light_arcs].sum()) == 0
    assert bool((cover[g.light_arcs:] == 1).all())


def test_split_is_the_default_resident_layout_and_bit_stable():
    k = 50
    src, dst, w, y, n = _graph(18, 3_000_000, k, True, seed=3)
    g = DeviceGraph.from_edges(src, dst, w, n, device=DEV, pull=True)
    g.prepare_hot(k, enable=True)
    emb = Embedder(n, k, DEV)
    z = emb.embed(g, y, variant="pull")
    assert g.split and g.n_tails > 0
    assert torch.equal(z, emb.embed(g, y, variant="pull"))
    exp = oracle.serial_embed(src.cpu().numpy(), dst.cpu().numpy(), w.cpu().numpy(), y.cpu().numpy(), n, k)
    assert rel_err(z.cpu().numpy(), exp) <= 1e-4
