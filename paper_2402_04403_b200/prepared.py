"""Prepared graphs: graph preparation once, then the edge pass per call.

The reference keeps graph construction (``build_csr``) out of its timed
region and passes the stored ``CsrGraph`` to ``embed_parallel`` on every call
(bench.py:1-7, 84-86 there; encoder.py:123-194).  ``prepare`` is that
split for the GPU path: it turns a stored ``CsrGraph`` (or an ``EdgeList``)
into the pull layout once -- symmetric CSR, hot-label tier, rows sorted by
slot and padded to 8 arcs -- and ``embed_parallel(prepared, y, out=...)``
then runs only the per-call work:

* ``residency="host"`` (default): the prepared layout sits in pinned host
  memory, packed (``stream.HostPipeline``); each call copies the labels and
  the graph in row chunks, runs the histogram and the chunked pull, and
  copies Z out row-sparse into the caller's host array, with the copies,
  the kernels and the host-side expansion overlapping.  HBM only holds two
  chunks, so graphs larger than device memory work the same way.
* ``residency="device"``: the layout stays in HBM; each call runs the
  histogram and the pull and delivers Z where ``out`` lives: into a CUDA
  tensor through one replay of the pass recorded as a CUDA graph, into host
  memory row-sparse per chunk (labels in, compacted Z out, host-side
  expansion overlapping), as the streamed path does minus the graph copy.

Host buffers passed as ``out`` (or as the labels) are page-locked with
``cudaHostRegister`` on first use and kept registered while the prepared
graph lives (``close()`` releases them), so repeated calls with the same
buffer -- what the reference's bench does with ``out=`` -- copy straight
into it.
"""

import logging
import time

import numpy as np

from .errors import ValidationError
from .graph import CsrGraph, EdgeList, _is_torch

logger = logging.getLogger(__name__)


class PreparedGraph:
    """A graph prepared for repeated edge passes with ``k`` classes.

    Attributes: ``n``, ``k``, ``s`` (listed edges), ``directed``,
    ``residency``, ``prep_s`` (seconds per preparation step), ``variant``
    (always "pull": the prepared layout is the exact integer pull).
    """

    MAX_REGISTERED = 8

    def __init__(self):
        self.n = self.k = self.s = 0
        self.directed = True
        self.residency = "host"
        self.prep_s = {}
        self.variant = "pull"
        self.device = None
        self._dg = None  # residency="device": the DeviceGraph
        self._pipe = None  # residency="host": the HostPipeline
        self._pipe_res = None  # residency="device", host results: HostPipeline over the resident graph
        self._chunks = 32
        self._emb = None
        self._graph = None  # residency="device": the pass recorded as a CUDA graph
        self._lab_buf = self._z_buf = None
        self._registered = {}  # (ptr, nbytes) -> (array kept alive, torch view)
        self.layout = "rows"  # "tiles": heavy rows regrouped by slot tile (device results only)
        self._closed = False

    # ------------------------------------------------------------ buffers
    def _register(self, arr):
        """A torch CPU view of host array ``arr`` that CUDA treats as pinned
        (cudaHostRegister once per buffer, cached)."""
        import torch

        t = arr if _is_torch(arr) else torch.from_numpy(arr)
        if t.is_pinned():
            return t
        key = (t.data_ptr(), t.numel() * t.element_size())
        hit = self._registered.get(key)
        if hit is not None:
            return hit[1]
        if len(self._registered) >= self.MAX_REGISTERED:
            old_key = next(iter(self._registered))
            torch.cuda.cudart().cudaHostUnregister(old_key[0])
            del self._registered[old_key]
        rc = torch.cuda.cudart().cudaHostRegister(key[0], key[1], 0)
        if int(rc) != 0:
            raise ValidationError(f"cudaHostRegister of a {key[1]}-byte host buffer failed ({int(rc)})")
        self._registered[key] = (arr, t)
        return t

    def close(self):
        """Unregister the host buffers and free the prepared layout."""
        if self._closed:
            return
        import torch

        for key in list(self._registered):
            torch.cuda.cudart().cudaHostUnregister(key[0])
        self._registered.clear()
        for pipe in (self._pipe, self._pipe_res):
            if pipe is not None:
                pipe.arena.close()
        self._dg = self._pipe = self._pipe_res = self._emb = None
        self._graph = self._lab_buf = self._z_buf = None
        self._closed = True

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --------------------------------------------------------------- pass
    def run(self, y, out=None, inv=None):
        """One edge pass (the body of embed_parallel for a prepared graph)."""
        import torch

        from .device import to_device

        if self._closed:
            raise ValidationError("prepared graph is closed")
        if y.n != self.n:
            raise ValidationError(f"graph has {self.n} nodes but labels have {y.n}")
        if y.k != self.k:
            raise ValidationError(f"graph was prepared for k={self.k} but labels have k={y.k}")
        host_result = (out is not None and not (_is_torch(out) and out.is_cuda)) or \
            (out is None and not (_is_torch(y.labels) and y.labels.is_cuda))
        if self.residency == "device" and not host_result:
            if inv is None:
                # the pass is recorded once as a CUDA graph and replayed on
                # the new labels: one host launch per call (small graphs are
                # launch-bound: C1 0.094 -> 0.019 ms)
                if self._graph is None:
                    self._lab_buf = torch.empty(self.n, dtype=torch.int32, device=self.device)
                    self._z_buf = torch.empty((self.n, self.k), dtype=torch.float32, device=self.device)
                    self._lab_buf.copy_(to_device(y.labels, torch.int32, self.device))
                    self._graph = self._emb.capture(self._dg, self._lab_buf, self._z_buf)
                else:
                    self._lab_buf.copy_(to_device(y.labels, torch.int32, self.device), non_blocking=True)
                    self._graph.replay()
                z_d = self._z_buf if (out is not None and not _is_torch(out)) else self._z_buf.clone()
            else:
                lab_d = to_device(y.labels, torch.int32, self.device)
                z_d = out if (_is_torch(out) and out.is_cuda) else None
                z_d = self._emb.embed(self._dg, lab_d, variant="pull", z=z_d, inv=inv)
            torch.cuda.current_stream(self.device).synchronize()
            if out is None:
                return z_d if (_is_torch(y.labels) and y.labels.is_cuda) else z_d.cpu().numpy()
            if _is_torch(out):
                if out.data_ptr() != z_d.data_ptr():
                    out.copy_(z_d)
                return out
            out[...] = z_d.cpu().numpy()
            return out
        # host result: labels and Z through pinned host memory -- the graph
        # streamed from pinned host memory (host residency) or read where it
        # lies in HBM (device residency), Z copied out row-sparse per chunk
        pipe = self._pipe
        if self.residency == "device" and self.layout == "tiles":
            raise ValidationError("a prepared graph with layout='tiles' delivers Z to CUDA tensors only "
                                  "(pass device labels / out=, or prepare with layout='rows')")
        if self.residency == "device":
            if self._pipe_res is None:
                from .stream import HostPipeline

                self._pipe_res = HostPipeline(self._dg, self.k, chunks=self._chunks, device=self.device,
                                              resident=True)
            pipe = self._pipe_res
        lab = y.labels
        if _is_torch(lab):
            lab = lab.cpu() if lab.is_cuda else lab
            h_y = lab.to(torch.int32).contiguous()
            h_y = h_y if h_y.is_pinned() else self._register(h_y)
        else:
            h_y = self._register(np.ascontiguousarray(lab, dtype=np.int32))
        target = out
        if out is None:
            h_z = torch.empty((self.n, self.k), dtype=torch.float32).pin_memory()
            result = h_z.numpy()
        elif _is_torch(out) and not out.is_cuda and out.dtype == torch.float32:
            h_z = out if out.is_pinned() else self._register(out)
            result = out
        elif isinstance(out, np.ndarray) and out.dtype == np.float32:
            h_z = self._register(out)
            result = out
        else:  # float64 host array or a CUDA tensor: through a pinned f32 Z
            h_z = torch.empty((self.n, self.k), dtype=torch.float32).pin_memory()
            result = None
        pipe.run(h_y, h_z, self._emb, inv=inv)
        if result is not None:
            return result
        if _is_torch(target):
            target.copy_(h_z)
        else:
            target[...] = h_z.numpy()
        return target

    @property
    def h2d_bytes_per_call(self):
        """Bytes one host-result call copies in (labels, and for host
        residency the graph chunks and the hot tier)."""
        pipe = self._pipe if self._pipe is not None else self._pipe_res
        if pipe is None:
            return 0
        import torch

        return pipe.h2d_bytes(torch.empty(self.n, dtype=torch.int32))

    @property
    def d2h_bytes_last_call(self):
        pipe = self._pipe if self._pipe is not None else self._pipe_res
        return 0 if pipe is None else int(pipe.d2h_bytes)


STREAM_CHUNKS = 96    # row chunks of a call that streams the prepared graph from pinned host memory
RESIDENT_CHUNKS = 32  # ... of a call on a graph resident in HBM (only Z crosses PCIe)


def prepare(g, k, *, device=None, residency="host", chunks=None, accounting=None, layout="rows"):
    """Prepare ``g`` (a ``CsrGraph`` or an ``EdgeList``) for repeated edge
    passes with ``k`` classes; returns a ``PreparedGraph`` that
    ``embed_parallel`` accepts in place of the graph.

    Preparation -- upload, symmetric CSR, hot-label plan, row sort and pad,
    and (host residency) packing into pinned host memory -- happens here,
    once; ``prepared.prep_s`` times each step.  The prepared layout is the
    exact integer pull: weights whose range fails its fixed-point gate raise
    ``ValidationError`` (call ``embed_parallel(g, y)`` for the push then).

    ``layout="tiles"`` (device residency only) also regroups the heavy rows'
    targets by label-table tile (``DeviceGraph.tile_heavy``: their lookups
    then hit shared memory; C4 19.5 -> 18.3 ms per pass, same Z bits).  Such
    a prepared graph delivers Z to CUDA tensors only: the host-result path
    reads the graph in row chunks, which the regrouped layout does not have.

    ``chunks``: row chunks a host-result call streams (default: 96 when the
    graph is streamed from host memory, 32 when it is resident in HBM; C4
    streamed 24 / 32 / 48 / 64 / 96 / 128 / 192 chunks: 397 / 389 / 389 /
    379 / 372 / 376 / 379 ms, resident 32 / 96: 230 / 237 ms).
    """
    import torch

    from .device import PULL_REL_ERR_MAX, DeviceGraph, Embedder, require_cuda
    from .encoder import EdgeAccounting, edge_accounting

    if residency not in ("host", "device"):
        raise ValidationError("residency must be 'host' or 'device'")
    if layout not in ("rows", "tiles"):
        raise ValidationError("layout must be 'rows' or 'tiles'")
    if layout == "tiles" and residency != "device":
        raise ValidationError("layout='tiles' needs residency='device'")
    k = int(k)
    if k < 1:
        raise ValidationError("class count k must be positive")
    if chunks is None:
        chunks = STREAM_CHUNKS if residency == "host" else RESIDENT_CHUNKS
    if chunks < 1:
        raise ValidationError("chunks must be at least 1")
    dev = require_cuda(device)
    p = PreparedGraph()
    p.k, p.device, p.residency, p._chunks = k, dev, residency, chunks
    t0 = time.perf_counter()
    if isinstance(g, EdgeList):
        p.n, p.s, p.directed = g.n, g.s, g.directed
        dg = DeviceGraph.from_edges(g.src, g.dst, g.w, g.n, device=dev, pull=True)
    elif isinstance(g, CsrGraph):
        if accounting is None:
            accounting = edge_accounting(g)
        symmetric = accounting is EdgeAccounting.SOURCE_ONLY
        p.n, p.directed = g.n, not symmetric
        dg = DeviceGraph.from_csr(g.offsets, g.targets, g.weights, g.n, symmetric, device=dev, pull=True)
        p.s = dg.s
    else:
        raise ValidationError("prepare() takes a CsrGraph or an EdgeList")
    torch.cuda.synchronize(dev)
    p.prep_s["csr"] = time.perf_counter() - t0
    if dg.weighted and dg.rel_err > PULL_REL_ERR_MAX:
        raise ValidationError(
            f"weights span too wide a range for the exact fixed-point pull (rounding bound {dg.rel_err:.2e}); "
            f"call embed_parallel(g, y) on the stored graph (push variant)")
    t0 = time.perf_counter()
    dg.prepare_hot(k)
    torch.cuda.synchronize(dev)
    p.prep_s["hot_sort_pad"] = time.perf_counter() - t0
    p._emb = Embedder(p.n, k, dev)
    if residency == "device":
        if layout == "tiles":
            t0 = time.perf_counter()
            p.layout = "tiles" if dg.tile_heavy() else "rows"
            torch.cuda.synchronize(dev)
            p.prep_s["tile_heavy"] = time.perf_counter() - t0
        p._dg = dg
        return p
    from .stream import HostPipeline

    t0 = time.perf_counter()
    p._pipe = HostPipeline(dg, k, chunks=chunks, device=dev)
    del dg
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()
    p.prep_s["pack_pin"] = time.perf_counter() - t0
    return p


__all__ = ["PreparedGraph", "prepare"]
