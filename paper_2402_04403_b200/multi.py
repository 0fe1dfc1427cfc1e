"""Row-range sharding over the GPUs of one process (the CLI's ``--gpus N``).

The same scheme as bench.py's one-process-per-GPU run (shard.py, SURVEY.md
section 8(e) scheme 1), driven from one host process: shard i owns the node
rows [b_i, b_{i+1}) planned by shard.plan_rows, builds the symmetric CSR of
those rows on its device, runs histogram + pull there and copies its Z rows
into the caller's host array.  There is no cross-device traffic: every Z
row is written exactly once by its owner, so the result is bit-identical
to the single-GPU pull.  One host thread per device; shards that share a
device (``devices`` shorter than ``shards``) run one after another on it,
which is how the tests cover the N-shard path on a one-GPU box.
"""

import logging
import threading

import numpy as np

from .errors import ValidationError
from .graph import CsrGraph, EdgeList, _is_torch
from .labeling import LabelVector

logger = logging.getLogger(__name__)


def _shard_from_edges(el, n, shards, i, k, dev):
    import torch

    from .device import to_device
    from .shard import build_row_shard

    src = to_device(el.src, torch.int32, dev)
    dst = to_device(el.dst, torch.int32, dev)
    w = to_device(el.w, torch.float32, dev)
    return build_row_shard(src, dst, w, n, shards, i, k=k)


def _shard_from_symmetric_csr(g, bounds, i, dev):
    """Rows [lo, hi) of a symmetric (SOURCE_ONLY) CsrGraph are already the
    pull layout of that shard: slice them, keep global degrees for the hot plan."""
    import torch

    from .device import DeviceGraph, to_device

    lo, hi = int(bounds[i]), int(bounds[i + 1])
    off = g.offsets
    a0, a1 = int(off[lo]), int(off[hi])
    off_d = to_device(off, torch.int64, dev)
    local = (off_d[lo:hi + 1] - a0).contiguous()
    tgt = to_device(g.targets[a0:a1], torch.int32, dev)
    w = None if g.weights is None else to_device(g.weights[a0:a1], torch.float32, dev)
    dg = DeviceGraph.from_csr(local, tgt, w, hi - lo, True, device=dev)
    dg.n_nodes = g.n
    dg.global_offsets = off_d
    return dg, lo, hi


class ShardedPass:
    """Prepared row shards of one graph over a list of devices.

    prepare (constructor): plan rows, build each shard's pull layout and
    hot tier on its device, upload the labels -- graph preparation, outside
    any timed region as the reference keeps build_csr out (bench.py:1-7).
    run(): one edge pass (histogram + pull) on every shard, one host thread
    per device; returns per-device elapsed milliseconds (CUDA events on each
    device's launching stream).  gather(): the (n, k) Z on the host.
    """

    def __init__(self, graph, y: LabelVector, shards, devices=None):
        import torch

        from .device import Embedder, to_device
        from .shard import merge_weight_stats, plan_rows

        if shards < 1:
            raise ValidationError("shards must be at least 1")
        if devices is None:
            avail = torch.cuda.device_count()
            if shards > avail:
                raise ValidationError(f"requested {shards} GPUs but {avail} are visible")
            devices = list(range(shards))
        self.devices = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
        n, k = graph.n, y.k
        if n != y.n:
            raise ValidationError(f"graph has {n} nodes but labels have {y.n}")
        self.n, self.k, self.shards = n, k, shards
        self.s = graph.s if isinstance(graph, EdgeList) else (graph.s if graph.directed else graph.s // 2)
        symmetric = isinstance(graph, CsrGraph) and not graph.directed
        if isinstance(graph, CsrGraph) and graph.directed:
            # one arc per listed edge: the arcs are the listed edges
            off = graph.offsets.cpu().numpy() if _is_torch(graph.offsets) else graph.offsets
            rows = np.repeat(np.arange(n, dtype=np.int32), np.diff(off))
            graph = EdgeList(n=n, src=rows, dst=graph.targets, w=graph.weights, directed=True)
        bounds = None
        if symmetric and n:
            off = graph.offsets.cpu().numpy() if _is_torch(graph.offsets) else graph.offsets
            bounds = plan_rows(off, shards, k, graph.weights is not None)
        self.by_dev = {}
        for i in range(shards):
            self.by_dev.setdefault(self.devices[i % len(self.devices)], []).append(i)
        self.parts = {}  # shard -> (DeviceGraph, Embedder, labels_d, z_d, lo, hi)
        self.weighted = graph.weights is not None if isinstance(graph, CsrGraph) else graph.w is not None
        if n == 0:
            return

        def prep(dev, mine):
            torch.cuda.set_device(dev)
            lab = to_device(y.labels, torch.int32, dev)
            for i in mine:
                if symmetric:
                    g, lo, hi = _shard_from_symmetric_csr(graph, bounds, i, dev)
                else:
                    g, lo, hi = _shard_from_edges(graph, n, shards, i, k, dev)
                z = torch.empty((hi - lo, k), dtype=torch.float32, device=dev)
                self.parts[i] = (g, Embedder(n, k, dev), lab, z, lo, hi)
            torch.cuda.synchronize(dev)

        self._each_device(prep)
        # one fixed-point exponent for the whole graph: bit-identical to the
        # single-GPU pull
        stats = merge_weight_stats(p[0].weight_stats() for p in self.parts.values())
        for p in self.parts.values():
            p[0].adopt_scale(stats)
        # the merged weight range can fail the exact pull's fixed-point gate
        # even when no single shard does: then every shard pushes its own
        # rows' arcs (SOURCE_ONLY over the row shard, fp32 atomics into its
        # own Z rows; still no cross-device traffic)
        from .device import PULL_REL_ERR_MAX

        worst = max((p[0].rel_err for p in self.parts.values() if p[0].weighted), default=0.0)
        self.variant = "push" if worst > PULL_REL_ERR_MAX else "pull"
        if self.variant == "push":
            logger.warning("weights span too wide a range for the exact fixed-point pull over the whole graph "
                           "(rounding bound %.2e): the row shards run the push variant", worst)

        def finish(dev, mine):
            torch.cuda.set_device(dev)
            for i in mine:
                g, emb, lab, z, lo, hi = self.parts[i]
                if self.variant == "push":
                    g.to_source_only_coo()
                    emb.project(lab)  # validates the labels once
                else:
                    g.prepare_hot(k)
                    g.tile_heavy()  # repeated passes: heavy rows' targets regrouped by slot tile
                    emb.project(lab, g=g)  # validates the labels once
            torch.cuda.synchronize(dev)

        self._each_device(finish)

    def _each_device(self, fn):
        errors = []

        def wrap(dev, mine):
            try:
                fn(dev, mine)
            except BaseException as exc:  # re-raised on the caller's thread
                errors.append(exc)

        threads = [threading.Thread(target=wrap, args=(d, m)) for d, m in self.by_dev.items()]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]

    def run(self):
        """One edge pass on every shard; returns {device: elapsed ms}."""
        import torch

        elapsed = {}
        if self.n == 0:
            return elapsed

        def go(dev, mine):
            torch.cuda.set_device(dev)
            stream = torch.cuda.current_stream(dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for i in mine:
                g, emb, lab, z, _, _ = self.parts[i]
                if self.variant == "push":
                    emb.project(lab, validate=False)
                    emb.push(g, z)
                else:
                    emb.project(lab, validate=False, g=g)
                    emb.pull(g, z)
            b.record(stream)
            b.synchronize()
            elapsed[dev] = a.elapsed_time(b)

        self._each_device(go)
        return elapsed

    def gather(self):
        z = np.zeros((self.n, self.k), dtype=np.float32)
        for g, emb, lab, zi, lo, hi in self.parts.values():
            z[lo:hi] = zi.cpu().numpy()
        return z


def embed_sharded(graph, y: LabelVector, shards, devices=None):
    """Pull edge pass with the rows split over `shards` row ranges.

    graph    EdgeList (listed edges, both updates) or CsrGraph (directed
             storage is expanded to its listed edges; symmetric storage is
             sliced by rows)
    devices  CUDA devices to place shard i on devices[i % len(devices)]
             (default: 0..shards-1, which must all exist)
    Returns the (n, k) float32 Z as a numpy array.
    """
    sp = ShardedPass(graph, y, shards, devices)
    sp.run()
    return sp.gather()
