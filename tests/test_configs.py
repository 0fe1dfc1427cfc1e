"""Parity on the BASELINE.json configurations.

* C1 and C2 at full size, C3 / C4 / C5 at reduced size: the full f64 oracle
  (oracle.serial_embed, the reference's serial_pass rule) against the pull
  and the push; the pull is bit-stable; class counts are exact.
* C3, C4 and C5 at FULL size: a row sample (uniform rows plus the
  highest-degree hubs) against the C oracle's threaded
  sampled-row restatement of serial_pass (oracle.sampled_rows_par, pinned to
  oracle.serial_embed in tests/test_oracle.py), plus per-column mass
  accounting (sum_x Z[x,c] = inv[c] * sum over edges of w * ([Y[v]=c] +
  [Y[u]=c])).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from conftest import rel_err  # noqa: E402

from paper_2402_04403_b200 import synth  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph, Embedder  # noqa: E402

TOL = 1e-4
DEV = torch.device("cuda")


def _pull_push(src, dst, w, y, n, k):
    g = DeviceGraph.from_edges(src, dst, w, n, device=DEV, pull=True, keep_coo=True)
    emb = Embedder(n, k, DEV)
    zp = emb.embed(g, y, variant="pull")
    zp2 = emb.pull(g).clone()
    zq = emb.embed(g, y, variant="push")
    counts = emb.counts.cpu().numpy()
    return zp, zp2, zq, counts


@pytest.mark.parametrize("idx,override", [
    (1, {}),
    (2, {}),
    (3, {"scale_override": 19}),
    (4, {"scale_override": 19}),
    (5, {"edges_override": 6_400_000}),
], ids=["C1", "C2", "C3-s19", "C4-s19", "C5-n1e5"])
def test_config_full_oracle(idx, override):
    src, dst, w, y, n, k, directed = synth.make_config(idx, **override)
    zp, zp2, zq, counts = _pull_push(src, dst, w, y, n, k)
    yh = y.cpu().numpy()
    assert np.array_equal(counts, np.bincount(yh, minlength=k + 1))
    exp = oracle.serial_embed(src.cpu().numpy(), dst.cpu().numpy(), None if w is None else w.cpu().numpy(), yh, n, k)
    assert torch.equal(zp, zp2), "pull is not run-to-run bit-stable"
    assert rel_err(zp.cpu().numpy(), exp) <= TOL
    assert rel_err(zq.cpu().numpy(), exp) <= TOL


def _sample_rows(src, dst, n, seed, uniform=65536, hubs=1024):
    gen = torch.Generator(device=DEV).manual_seed(seed)
    deg = torch.bincount(src.long(), minlength=n) + torch.bincount(dst.long(), minlength=n)
    top = torch.topk(deg, min(hubs, n)).indices
    rows = torch.unique(torch.cat([torch.randint(0, n, (uniform,), device=DEV, generator=gen), top]))
    return rows


@pytest.mark.parametrize("idx", [3, 4, 5], ids=["C3-full", "C4-full", "C5-full"])
def test_config_full_size_sampled(idx):
    """BASELINE sizes (C3: 268M undirected edges, K=100, 10% labeled; C4:
    1.8e9 directed weighted edges, K=50; C5: n=4e6, 256M edges, K=1000):
    the pull's Z on >= 65K uniform rows plus the 1024 highest-degree rows
    against the pinned C oracle's sampled-row restatement of serial_pass
    (oracle.sampled_rows_par, f64), and every column's mass sum_x Z[x, c]
    against the oracle's mass accounting (reference test_parallel.py:54-64).
    Counts exact; pull run-to-run bit-stable."""
    src, dst, w, y, n, k, directed = synth.make_config(idx)
    g = DeviceGraph.from_edges(src, dst, w, n, device=DEV, pull=True)
    emb = Embedder(n, k, DEV)
    z = emb.embed(g, y, variant="pull")
    z2 = emb.pull(g)
    assert torch.equal(z, z2), "pull is not run-to-run bit-stable"
    del z2
    yh = y.cpu().numpy()
    assert np.array_equal(emb.counts.cpu().numpy(), np.bincount(yh, minlength=k + 1))
    del g
    torch.cuda.empty_cache()
    rows = _sample_rows(src, dst, n, idx, uniform=65536 if idx != 5 else 131072)
    zr = z[rows].cpu().numpy()
    col = sum(z[a:a + (1 << 22)].double().sum(0) for a in range(0, n, 1 << 22)).cpu().numpy()
    del z
    torch.cuda.empty_cache()
    src_h, dst_h = src.cpu().numpy(), dst.cpu().numpy()
    w_h = None if w is None else w.cpu().numpy()
    del src, dst, w
    zs, mass = oracle.sampled_rows_par(src_h, dst_h, w_h, yh, k, rows.cpu().numpy())
    assert rel_err(zr, zs) <= TOL
    assert np.allclose(col, mass, rtol=1e-5, atol=1e-9)
