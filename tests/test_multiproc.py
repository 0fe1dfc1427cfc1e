"""Multi-process sharding logic on CPU (gloo, world_size 2).

The device path of a shard is the single-GPU pull on a row range
(shard.build_row_shard); what multi-GPU adds is the partitioning and, for
edge-range sharding, the reduce-scatter.  Both are exercised here with the
oracle standing in for each rank's device pass:

* row-range: every rank plans the same bounds from the same offsets, takes
  its rows of the symmetric CSR and computes their Z rows with the
  SOURCE_ONLY rule; the gathered slices equal the full oracle Z.
* edge-range: every rank embeds its contiguous slice of the listed edges
  into a full partial Z; shard.reduce_scatter_rows leaves each rank its row
  slice of the sum.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2402_04403_b200 import shard

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _graph(seed, n=3000, s=20000, k=7):
    rng = np.random.default_rng(seed)
    # skewed sources so that an arc-balanced split differs from an even one
    src = (rng.pareto(1.5, s) * 50).astype(np.int64) % n
    dst = rng.integers(0, n, s)
    w = (1.0 - rng.random(s)).astype(np.float32).astype(np.float64)
    y = rng.integers(0, k + 1, n).astype(np.int64)
    return src, dst, w, y, n, k


def _worker(rank, port, seed, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        src, dst, w, y, n, k = _graph(seed)
        _, _, row = oracle.projection(y, k)
        full = oracle.serial_embed(src, dst, w, y, n, k)
        if mode == "scale":
            # every rank adopts the whole graph's fixed-point exponent
            from paper_2402_04403_b200.device import DeviceGraph

            g = DeviceGraph(10, 10, torch.device("cpu"))
            mine = [(12.5, 0.75, 1e-3), (3.0, 0.999, 2e-6)][rank]
            g.max_row_abs, g.max_abs, g.min_abs = mine
            g.adopt_scale(mine)
            own = g.scale_exp
            shard.unify_scale_distributed(g)
            ref = DeviceGraph(10, 10, torch.device("cpu"))
            ref.adopt_scale(shard.merge_weight_stats([(12.5, 0.75, 1e-3), (3.0, 0.999, 2e-6)]))
            assert g.scale_exp == ref.scale_exp <= own and g.rel_err == ref.rel_err
            q.put((rank, "ok", g.scale_exp))
        elif mode == "rows":
            off, tgt, wts = oracle.build_csr(src, dst, w, n, directed=False)  # symmetric CSR
            bounds = shard.plan_rows(off, WORLD, k, weighted=True)
            got = [torch.zeros(WORLD + 1, dtype=torch.int64) for _ in range(WORLD)]
            dist.all_gather(got, torch.from_numpy(bounds))
            assert all(torch.equal(g, got[0]) for g in got), "ranks disagree on the plan"
            lo, hi = int(bounds[rank]), int(bounds[rank + 1])
            loc_off = off[lo:hi + 1] - off[lo]
            a, b = int(off[lo]), int(off[hi])
            z = oracle.parallel_embed(loc_off, tgt[a:b], wts[a:b], y, k, False, 1,
                                      row_value=row, label32=y.astype(np.int32))
            np.testing.assert_allclose(z, full[lo:hi], rtol=1e-12, atol=1e-15)
            # the slices tile [0, n) exactly
            sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(WORLD)]
            dist.all_gather(sizes, torch.tensor([hi - lo]))
            assert sum(int(x) for x in sizes) == n
            q.put((rank, "ok", hi - lo))
        else:
            e = shard.plan_edges(src.size, WORLD)
            a, b = int(e[rank]), int(e[rank + 1])
            part = oracle.serial_embed(src[a:b], dst[a:b], w[a:b], y, n, k)
            mine = shard.reduce_scatter_rows(torch.from_numpy(part), WORLD)
            per = -(-n // WORLD)
            lo, hi = rank * per, min(n, (rank + 1) * per)
            np.testing.assert_allclose(mine[:hi - lo].numpy(), full[lo:hi], rtol=1e-12, atol=1e-15)
            assert not mine[hi - lo:].any()  # padding rows stay zero
            q.put((rank, "ok", hi - lo))
    except Exception as ex:  # pragma: no cover - reported to the parent
        q.put((rank, f"fail: {type(ex).__name__}: {ex}", 0))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["rows", "edges", "scale"])
def test_sharding_world2_gloo(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, 11, mode, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get(timeout=10) for _ in range(WORLD))
    assert all(p.exitcode == 0 for p in procs), res
    assert all(r[1] == "ok" for r in res), res
    if mode == "rows":
        # arc-balanced: the skewed head gets fewer rows than an even split
        assert res[0][2] != res[1][2]


def test_plan_rows_balances_cost():
    src, dst, w, y, n, k = _graph(3, n=20000, s=200000, k=50)
    off, _, _ = oracle.build_csr(src, dst, w, n, directed=False)
    for world in (1, 2, 4, 8):
        b = shard.plan_rows(off, world, k, weighted=True)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
        cost = off[b] * 8 + b * 4 * k
        per = np.diff(cost)
        # within one row's worth of cost of the ideal share
        row_max = int(np.max(np.diff(off))) * 8 + 4 * k
        assert per.max() - per.min() <= 2 * row_max
    assert list(shard.plan_edges(10, 4)) == [0, 2, 5, 7, 10]


def _hist_worker(rank, port, q):
    # sharded histogram (bench.py row-range run): each rank counts its
    # contiguous n/world slice of the labels, one all-reduce of k+1 int64
    # gives np.bincount of the whole vector on every rank
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        rng = np.random.default_rng(5)
        n, k = 10_007, 13
        y = rng.integers(0, k + 1, n)
        lo, hi = shard.label_slice(n, WORLD, rank)
        counts = torch.from_numpy(oracle.bincount(y[lo:hi], k))
        shard.allreduce_counts(counts)
        assert np.array_equal(counts.numpy(), np.bincount(y, minlength=k + 1))
        spans = [torch.zeros(2, dtype=torch.int64) for _ in range(WORLD)]
        dist.all_gather(spans, torch.tensor([lo, hi]))
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(int(spans[i][1]) == int(spans[i + 1][0]) for i in range(WORLD - 1))
        q.put((rank, "ok", hi - lo))
    except Exception as ex:  # pragma: no cover
        q.put((rank, f"fail: {type(ex).__name__}: {ex}", 0))
        raise
    finally:
        dist.destroy_process_group()


def test_sharded_histogram_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hist_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get(timeout=10) for _ in range(WORLD))
    assert all(p.exitcode == 0 for p in procs), res
    assert all(r[1] == "ok" for r in res), res
    assert shard.label_slice(10, 4, 3) == (7, 10)


def _extra_steps_worker(rank, port, q):
    # bench.py after the timed region: every rank runs the SAME number of
    # untimed steps (a step holds collectives), derived from the slowest
    # rank's step time, whatever its own clock says
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import importlib.util

        spec = importlib.util.spec_from_file_location(
            "bench_mod", os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "bench.py"))
        bench = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(bench)
        mine = [90.0, 250.0][rank]  # ms over 10 timed steps: 9 and 25 ms per step
        count = bench.extra_steps(mine, 10, WORLD)
        counts = [torch.zeros(1, dtype=torch.int64) for _ in range(WORLD)]
        dist.all_gather(counts, torch.tensor([count]))
        assert int(counts[0]) == int(counts[1]) == 40, counts
        # the steps' collectives then match: WORLD ranks, `count` all-reduces each
        t = torch.ones(1)
        for _ in range(count):
            dist.all_reduce(t)
        q.put((rank, "ok", count))
    except Exception as ex:  # pragma: no cover
        q.put((rank, f"fail: {type(ex).__name__}: {ex}", 0))
        raise
    finally:
        dist.destroy_process_group()


def test_bench_extra_steps_agree_across_ranks_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_extra_steps_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get(timeout=10) for _ in range(WORLD))
    assert all(p.exitcode == 0 for p in procs), res
    assert all(r[1] == "ok" for r in res), res
