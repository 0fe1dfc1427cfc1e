"""Tile-major heavy region (DeviceGraph.tile_heavy, csrc/gee_tiles.cu): the
relocated layout gives the row-major pull's Z bit for bit and stays within
the parity bar against the f64 oracle."""

import numpy as np
import pytest

import oracle
from conftest import rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2402_04403_b200 import synth  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph, Embedder  # noqa: E402

TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _hub_graph(seed, n, weighted, signed=False, mega=False):
    """R-MAT-like skew by hand: a few hubs (one above 65536 arcs when `mega`:
    several work items), a dense cluster and a random background."""
    rng = np.random.default_rng(seed)
    parts_s, parts_d = [], []
    hubs = [0, 3, n - 1, n // 2]
    degs = [150_000 if mega else 30_000, 9_000, 5_000, 2_500]
    for h, d in zip(hubs, degs):
        parts_s.append(np.full(d, h, np.int64))
        parts_d.append((rng.random(d) ** 3 * n).astype(np.int64))  # skewed toward low ids
    parts_s.append(rng.integers(0, n, 60_000))
    parts_d.append(rng.integers(0, n, 60_000))
    parts_s.append(rng.integers(0, 64, 20_000))
    parts_d.append(rng.integers(0, 64, 20_000))
    src, dst = np.concatenate(parts_s), np.concatenate(parts_d)
    w = None
    if weighted:
        w = (1.0 - rng.random(src.size)).astype(np.float32)
        if signed:
            w = (w * rng.choice([-1.0, 1.0], src.size)).astype(np.float32)
    return src, dst, w


def _pull_both(src, dst, w, y, n, k, hot, tile_slots, max_tiles):
    dev = "cuda:0"
    zs = []
    for tiles in (False, True):
        g = DeviceGraph.from_edges(torch.as_tensor(src, dtype=torch.int32), torch.as_tensor(dst, dtype=torch.int32),
                                   None if w is None else torch.as_tensor(w), n, device=dev, pull=True)
        g.prepare_hot(k, enable=hot)
        assert g.n_heavy >= 3
        if tiles:
            assert g.tile_heavy(tile_slots=tile_slots, max_tiles=max_tiles)
            assert g.heavy_layout == "tiles" and g.n_items >= g.n_heavy
            lens = (g.offsets[1:] - g.offsets[:-1])
            assert int(lens[g.heavy_rows.long()].sum()) == 0
        emb = Embedder(n, k, device=dev)
        emb.project(torch.as_tensor(y, dtype=torch.int32, device=dev), g=g)
        z1 = emb.pull(g).clone()
        z2 = emb.pull(g)
        assert torch.equal(z1, z2), "not bit-stable"
        zs.append(z1.cpu().numpy())
    return zs


@pytest.mark.parametrize("hot", [True, False])
@pytest.mark.parametrize("weighted,signed", [(True, False), (False, False), (True, True)])
@pytest.mark.parametrize("tile_slots,max_tiles", [(256, 8), (4096, 3), (1024, 1000)])
def test_tiles_match_row_layout_bitwise(hot, weighted, signed, tile_slots, max_tiles):
    n, k = 20_000, 50
    src, dst, w = _hub_graph(11, n, weighted, signed)
    y = synth.uniform_labels_numpy(n, k, seed=3)
    z_rows, z_tiles = _pull_both(src, dst, w, y, n, k, hot, tile_slots, max_tiles)
    assert np.array_equal(z_rows.view(np.uint32), z_tiles.view(np.uint32))
    exp = oracle.serial_embed(src, dst, w, np.asarray(y, dtype=np.int64), n, k)
    if not signed:
        assert rel_err(z_tiles, exp) <= TOL


@pytest.mark.parametrize("short", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("k", [1, 3, 50])
def test_short_rows_skip_the_windows_bitwise(monkeypatch, short, k):
    """Weighted rows of at most SHORT_ROW_ARCS arcs are reduced in registers
    by the lane that holds them (gee_reduce_blocks_short): same bits as the
    windows for every threshold, with repeated classes (k = 1, 3), signed
    weights that cancel, unlabeled targets and self-loops."""
    monkeypatch.setattr(DeviceGraph, "SHORT_ROW_ARCS", short)
    n = 40_000
    rng = np.random.default_rng(100 + short)
    src0, dst0, w0 = _hub_graph(23, n, True, signed=True)
    # a sparse background: most rows end up with 1-4 arcs
    s1, d1 = rng.integers(0, n, 30_000), rng.integers(0, n, 30_000)
    loops = rng.integers(0, n, 500)
    src = np.concatenate([src0, s1, loops, s1[:2000]])
    dst = np.concatenate([dst0, d1, loops, d1[:2000]])
    w1 = (1.0 - rng.random(s1.size)).astype(np.float32) * rng.choice([-1.0, 1.0], s1.size).astype(np.float32)
    w = np.concatenate([w0, w1, np.ones(500, np.float32), -w1[:2000]])  # the last 2000 cancel their twins
    y = rng.integers(0, k + 1, n)
    z_rows, z_tiles = _pull_both(src, dst, w, y, n, k, True, 1024, 8)
    assert np.array_equal(z_rows.view(np.uint32), z_tiles.view(np.uint32))
    exp = oracle.serial_embed(src, dst, w, y.astype(np.int64), n, k)
    big = np.abs(exp) > 1e-3 * np.abs(exp).max()
    assert np.max(np.abs(z_tiles[big] - exp[big]) / np.abs(exp[big])) <= TOL


@pytest.mark.parametrize("align", [16, 32, 48])
def test_span_alignment_changes_no_bits(monkeypatch, align):
    """(tile, row) spans padded to 16, 32 (the default: whole sectors of
    class bytes) or 48 arcs: same Z bits as the row-major layout."""
    monkeypatch.setattr(DeviceGraph, "SPAN_ALIGN", align)
    n, k = 20_000, 50
    src, dst, w = _hub_graph(41, n, True, signed=True)
    y = synth.uniform_labels_numpy(n, k, seed=13)
    z_rows, z_tiles = _pull_both(src, dst, w, y, n, k, True, 512, 6)
    assert np.array_equal(z_rows.view(np.uint32), z_tiles.view(np.uint32))


@pytest.mark.parametrize("k", [1, 7, 255])
def test_tiles_mega_rows_and_k(k):
    n = 30_000
    src, dst, w = _hub_graph(5, n, True, mega=True)
    y = np.random.default_rng(8).integers(0, k + 1, n)
    z_rows, z_tiles = _pull_both(src, dst, w, y, n, k, True, 512, 16)
    assert np.array_equal(z_rows.view(np.uint32), z_tiles.view(np.uint32))
    exp = oracle.serial_embed(src, dst, w, y.astype(np.int64), n, k)
    assert rel_err(z_tiles, exp) <= TOL


def test_tiles_default_tile_size_and_guards():
    """Default 192 KB tiles on a graph whose table spans two tiles; the Z
    rows around the heavy rows are not touched by the heavy reducer."""
    n, k = 300_000, 50
    src, dst, w = _hub_graph(2, n, True)
    y = np.random.default_rng(1).integers(0, k + 1, n)
    z_rows, z_tiles = _pull_both(src, dst, w, y, n, k, True, None, None)
    assert np.array_equal(z_rows.view(np.uint32), z_tiles.view(np.uint32))


def test_tile_heavy_is_a_noop_without_heavy_rows_or_for_wide_k():
    rng = np.random.default_rng(0)
    n = 2000
    src, dst = rng.integers(0, n, 5000), rng.integers(0, n, 5000)
    g = DeviceGraph.from_edges(torch.as_tensor(src, dtype=torch.int32), torch.as_tensor(dst, dtype=torch.int32), None,
                               n, device="cuda:0", pull=True)
    g.prepare_hot(5)
    assert g.n_heavy == 0 and not g.tile_heavy() and g.heavy_layout == "rows"
    src, dst, _ = _hub_graph(1, n, False)
    g = DeviceGraph.from_edges(torch.as_tensor(src, dtype=torch.int32), torch.as_tensor(dst, dtype=torch.int32), None,
                               n, device="cuda:0", pull=True)
    g.prepare_hot(300)
    assert g.n_heavy > 0 and not g.tile_heavy() and g.heavy_layout == "rows"


def test_tiles_random_battery():
    """Random shapes: tile sizes that do not divide the table, tiles reaching
    past the table's end, rows that live entirely in one tile or entirely in
    the tail, unlabeled vertices."""
    rng = np.random.default_rng(2024)
    for case in range(12):
        n = int(rng.integers(3000, 40_000))
        k = int(rng.choice([1, 3, 50, 63, 64, 200]))
        weighted = bool(rng.integers(0, 2))
        nh = int(rng.integers(3, 8))
        parts_s, parts_d = [], []
        for _ in range(nh):
            d = int(rng.integers(2100, 12_000))
            lo = int(rng.integers(0, n - 1))
            hi = int(rng.integers(lo + 1, n + 1)) if rng.random() < 0.5 else n
            parts_s.append(np.full(d, int(rng.integers(0, n)), np.int64))
            parts_d.append(rng.integers(lo, hi, d))
        parts_s.append(rng.integers(0, n, 30_000))
        parts_d.append(rng.integers(0, n, 30_000))
        src, dst = np.concatenate(parts_s), np.concatenate(parts_d)
        w = (2.0 * rng.random(src.size) - 0.5).astype(np.float32) if weighted else None
        y = np.where(rng.random(n) < 0.3, 0, rng.integers(1, k + 1, n))
        ts = int(rng.choice([16, 48, 1000 * 16, 4096, 65536]))
        mt = int(rng.choice([1, 2, 5, 1000]))
        z_rows, z_tiles = _pull_both(src, dst, w, y, n, k, bool(rng.integers(0, 2)), ts, mt)
        assert np.array_equal(z_rows.view(np.uint32), z_tiles.view(np.uint32)), (case, n, k, ts, mt)
