"""prepare() + embed_parallel(prepared, y, out=...): the public host-buffer
path (graph preparation once, the edge pass per call), against the stored
graph's own embed_parallel and the CPU oracle (reference encoder.py:123-194:
host CSR + labels in, host Z out, ``out=`` reused across calls)."""

import numpy as np
import pytest

import oracle
from conftest import rel_err

from paper_2402_04403_b200 import (CsrGraph, EdgeList, LabelVector, ProjectionMatrix, ValidationError,
                                   build_projection, embed_parallel, prepare)
from paper_2402_04403_b200.encoder import last_pass

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _graph(seed, n=3000, s=40_000, weighted=True, directed=True, signed=False):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, s).astype(np.int32)
    dst = (src + rng.zipf(1.6, s) % n).astype(np.int32) % n  # some hubs and locality
    src[: s // 50] = 3  # one heavy row
    w = None
    if weighted:
        w = rng.random(s) + 0.01
        if signed:
            w *= np.where(rng.random(s) < 0.5, -1.0, 1.0)
        w = w.astype(np.float32)
    return src, dst, w


def _csr(src, dst, w, n, directed):
    off, tgt, wts = oracle.build_csr(src, dst, w, n, directed)
    return CsrGraph(n=n, offsets=off, targets=tgt, weights=None if w is None else wts, directed=directed)


@pytest.mark.parametrize("directed", [True, False])
@pytest.mark.parametrize("weighted,signed", [(True, False), (True, True), (False, False)])
@pytest.mark.parametrize("residency", ["host", "device"])
def test_prepared_matches_stored_graph_and_oracle(directed, weighted, signed, residency):
    n, k = 3000, 13
    src, dst, w = _graph(7, n=n, weighted=weighted, signed=signed)
    y = LabelVector(labels=np.random.default_rng(8).integers(0, k + 1, n), k=k)
    g = _csr(src, dst, w, n, directed)
    p = prepare(g, k, residency=residency, chunks=3)
    assert p.n == n and p.k == k and p.s == src.size and p.directed == directed
    exp = oracle.serial_embed(src, dst, w, y.labels, n, k)
    ref = embed_parallel(g, y, variant="pull")
    out = np.full((n, k), np.nan, dtype=np.float32)
    for _ in range(2):  # out= reused (registered once), every entry rewritten
        got = embed_parallel(p, y, out=out)
        assert got is out
        assert last_pass()["reducer"] == "prepared"
        assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))
        out.fill(np.nan)
    fresh = embed_parallel(p, y)
    assert fresh.dtype == np.float32 and np.array_equal(fresh, ref)
    assert rel_err(fresh, exp) <= 1e-4
    z64 = np.empty((n, k))
    embed_parallel(p, y, out=z64)
    assert np.array_equal(z64, ref.astype(np.float64))
    p.close()
    with pytest.raises(ValidationError):
        embed_parallel(p, y)


def test_prepared_from_edge_list_and_device_labels():
    n, k = 2500, 9
    src, dst, w = _graph(11, n=n, s=30_000)
    el = EdgeList(n=n, src=src, dst=dst, w=w, directed=True)
    lab = np.random.default_rng(12).integers(0, k + 1, n)
    p = prepare(el, k, chunks=2)
    z_host = embed_parallel(p, LabelVector(labels=lab, k=k))
    z_dev = embed_parallel(p, LabelVector(labels=torch.as_tensor(lab, device="cuda"), k=k))
    assert np.array_equal(z_host, z_dev)
    out_d = torch.empty((n, k), dtype=torch.float32, device="cuda")
    embed_parallel(p, LabelVector(labels=lab, k=k), out=out_d)
    assert np.array_equal(out_d.cpu().numpy(), z_host)
    assert rel_err(z_host, oracle.serial_embed(src, dst, w, lab, n, k)) <= 1e-4


def test_prepared_projection_and_errors():
    n, k = 2000, 6
    src, dst, w = _graph(21, n=n, s=20_000)
    g = _csr(src, dst, w, n, True)
    lab = np.random.default_rng(22).integers(0, k + 1, n)
    y = LabelVector(labels=lab, k=k)
    p = prepare(g, k, chunks=2)
    proj = build_projection(y)
    scaled = ProjectionMatrix(n=n, k=k, row_value=proj.row_value * 2.0, label=proj.label)
    z = embed_parallel(p, y, projection=scaled)
    assert np.array_equal(z, embed_parallel(g, y, projection=scaled, variant="pull"))
    with pytest.raises(ValidationError, match="prepared for k=6"):
        embed_parallel(p, LabelVector(labels=lab, k=k + 1))
    with pytest.raises(ValidationError, match="nodes"):
        embed_parallel(p, LabelVector(labels=lab[:-1], k=k))
    with pytest.raises(ValidationError):
        embed_parallel(p, y, out=np.empty((n, k + 1), dtype=np.float32))
    with pytest.raises(ValidationError):
        embed_parallel(p, y, variant="push")
    with pytest.raises(ValidationError):
        embed_parallel(p, y, workers=0)
    wide = w.copy()
    wide[0] = 1e-30
    with pytest.raises(ValidationError, match="push"):
        prepare(_csr(src, dst, wide, n, True), k)


def test_device_residency_replays_one_graph_over_label_sets():
    # residency="device": CUDA labels -> the pass recorded as a CUDA graph on
    # the first call and replayed after; host labels / host out -> the
    # resident chunked pipeline (labels in, row-sparse Z out).  Every call
    # equals the stored graph's own pass.
    n, k = 3000, 11
    src, dst, w = _graph(31, n=n)
    g = _csr(src, dst, w, n, True)
    p = prepare(g, k, residency="device", chunks=8)  # chunk 5 leaves dense, the rest row-sparse
    rng = np.random.default_rng(32)
    for i in range(3):
        lab = rng.integers(0, k + 1, n)
        ref = embed_parallel(g, LabelVector(labels=lab, k=k), variant="pull")
        zd = embed_parallel(p, LabelVector(labels=torch.as_tensor(lab, device="cuda"), k=k))
        assert zd.is_cuda and np.array_equal(zd.cpu().numpy(), ref), i
        zh = embed_parallel(p, LabelVector(labels=lab, k=k))
        assert isinstance(zh, np.ndarray) and np.array_equal(zh, ref), i
    assert p._graph is not None and p._pipe_res is not None and p._pipe_res.resident
    assert p.h2d_bytes_per_call == n * 4  # only the labels cross PCIe


@pytest.mark.parametrize("residency", ["host", "device"])
@pytest.mark.parametrize("k", [1, 300])
def test_prepared_host_results_small_and_wide_k(k, residency):
    # k = 1 and the wide-K reducer (k > 255) through the streamed path and the
    # resident chunked path (7 chunks: chunk 5 leaves dense)
    n = 2500
    src, dst, w = _graph(41, n=n, s=25_000)
    g = _csr(src, dst, w, n, True)
    y = LabelVector(labels=np.random.default_rng(42).integers(0, k + 1, n), k=k)
    p = prepare(g, k, chunks=7, residency=residency)
    z = embed_parallel(p, y)
    assert np.array_equal(z, embed_parallel(g, y, variant="pull"))
    assert rel_err(z, oracle.serial_embed(src, dst, w, y.labels, n, k)) <= 1e-4


def test_device_residency_tile_layout_device_results_only():
    # layout="tiles": heavy rows' targets regrouped by slot tile; CUDA labels
    # in, CUDA Z out through the recorded pass; same bits as the stored
    # graph's pass.  Host results are refused (that path reads row chunks).
    n, k = 3000, 11
    src, dst, w = _graph(41, n=n, s=150_000)  # row 3 has 3000 arcs: one heavy row
    g = _csr(src, dst, w, n, True)
    p = prepare(g, k, residency="device", layout="tiles")
    assert p.layout == "tiles" and p._dg.heavy_layout == "tiles"
    rng = np.random.default_rng(42)
    out = torch.empty((n, k), dtype=torch.float32, device="cuda")
    for i in range(3):
        lab = rng.integers(0, k + 1, n)
        ref = embed_parallel(g, LabelVector(labels=lab, k=k), variant="pull")
        zd = embed_parallel(p, LabelVector(labels=torch.as_tensor(lab, device="cuda"), k=k), out=out)
        assert zd is out and np.array_equal(zd.cpu().numpy(), ref), i
    with pytest.raises(ValidationError, match="tiles"):
        embed_parallel(p, LabelVector(labels=lab, k=k))
    with pytest.raises(ValidationError, match="residency"):
        prepare(g, k, layout="tiles")
    with pytest.raises(ValidationError, match="layout"):
        prepare(g, k, residency="device", layout="columns")
    p.close()
