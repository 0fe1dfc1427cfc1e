"""Host-resident graph -> host Z, streamed through the GPU in row chunks.

A user of the reference calls ``embed_parallel(g, y)`` with a CSR graph and
labels in host memory and gets Z back in host memory (encoder.py:123-194).
With a graph of C4's size the PCIe copies dominate that call:
- about 31 GB of prepared CSR goes in;
- about 27 GB of Z comes out.

PCIe is full duplex, so this module overlaps the two. It splits the prepared
symmetric CSR into row chunks balanced by bytes. Then, on three CUDA streams:
- copy-in: H2D of chunk i+1 into one of two device slots;
- compute: the pull of chunk i (gather + block / heavy reduction), into one
  of two Z slots;
- copy-out: D2H of chunk i-1's Z rows into the caller's pinned host Z.

Events order the slot reuse, and each chunk's pull is exactly the
single-GPU pull on a row range (the same kernels as the row-range shards).

Z leaves the GPU row-sparse (``sparse=True``, the default): on C4 over 90%
of Z is zero, so each chunk is compacted on the device (gee_z_compact: u64
row masks, per-block offsets, packed nonzero values) and the host rebuilds
the dense rows in the caller's buffer with streaming stores
(gee_io_expand_rows, all host threads).  The compacted size is only known
once the chunk is computed, so the host issues each chunk's copy-out one
chunk behind the compute stream and expands two chunks behind; the copy-in
queue stays ahead of both.

The targets cross PCIe packed (``packed=True``, the default for the padded
layout): gee_pack_targets codes each chunk's slot-sorted targets as groups of
8 bit-width deltas at preparation time and its weights, without the row
padding, as lossless group fixed point (1-3 bytes per weight when the group's
weights are exact multiples of a common power of two, else raw f32; a chunk
whose groups all share one weight code sends that code instead of the
per-group bytes); gee_unpack_targets rebuilds the padded targets and weights
on the compute stream before the chunk's pull (C4: 31 GB of targets and
weights become about 18 GB; the rebuilt arrays are bit-identical, so Z is
too).

Graph preparation (CSR build, hot-label plan, per-chunk heavy-row items,
pinned host copies) happens once in ``HostPipeline(...)``. It is outside
the timed region, as the reference's ``build_csr`` is (bench.py:1-7 there).
"""

import ctypes
import threading

import numpy as np
import torch

from . import _lib
from .device import DeviceGraph, Embedder
from .errors import ValidationError
from .shard import plan_rows


class PinnedArena:
    """Page-locked host buffers of exact size: numpy memory registered with
    cudaHostRegister and released by close().  torch's pinned allocator
    rounds every block up to a power of two (a 9.3 GB payload would lock
    16 GB of host RAM) and .cpu().pin_memory() copies twice; the arena's
    buffers receive their device-to-host copy directly."""

    def __init__(self):
        self._held = []

    def empty(self, n, dtype=torch.uint8):
        itemsize = torch.empty(0, dtype=dtype).element_size()
        a = np.empty(max(1, n) * itemsize, dtype=np.uint8)
        rc = int(torch.cuda.cudart().cudaHostRegister(a.ctypes.data, a.nbytes, 0))
        if rc != 0:
            raise ValidationError(f"cudaHostRegister of {a.nbytes} bytes failed ({rc})")
        self._held.append(a)
        return torch.from_numpy(a).view(dtype)[:n]

    def copy_of(self, t):
        """A pinned host copy of tensor t (device or host)."""
        h = self.empty(t.numel(), t.dtype).view(t.shape) if t.numel() else torch.empty(0, dtype=t.dtype)
        if t.numel():
            h.copy_(t)
        return h

    def close(self):
        for a in self._held:
            torch.cuda.cudart().cudaHostUnregister(a.ctypes.data)
        self._held.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HostPipeline:
    """Streams a prepared graph held in pinned host memory through one GPU.

    ``resident=True``: the prepared graph stays in HBM (the caller keeps
    ``g`` alive); a call then only copies the labels in and the row-sparse Z
    out, chunk by chunk, with the same compaction and host-side expansion.
    """

    HOST_SLOTS = 3  # row-sparse Z chunks in host memory: one copying out while two expand
    DENSE_EVERY_STREAMED = 0  # streaming: the copy-in is the bound, no dense chunks
    # resident: 1 chunk in 8 copied out dense (C4 with the AVX-512 expansion: none 239-241, 12 251, 8 232-235,
    # 6 247-252, 4 266 ms; with the scalar expansion: none 298, 6 267, 4 273, 3 286, 2 338 ms)
    DENSE_EVERY_RESIDENT = 8
    # host threads rebuilding a chunk's dense rows (0: all).  Streaming, the
    # expansion's stores share host memory with the copy-in's DMA reads, so
    # fewer threads finish sooner (C4, AVX-512 expansion: 4 / 8 / 12 / 16
    # threads 571 / 387 / 419 / 434 ms); resident, the expansion is the bound
    # (4 / 8 / 12 / 16: 474 / 282 / 249 / 244 ms)
    EXPAND_THREADS_STREAMED = 8
    EXPAND_THREADS_RESIDENT = 0
    EXPAND_THREADS = None  # overrides both when set

    def __init__(self, g: DeviceGraph, k, chunks=16, device=None, packed=None, resident=False):
        if not g.has_pull or g.hot_k != k:
            raise ValidationError("HostPipeline needs a pull graph prepared for k (prepare_hot)")
        if g.heavy_layout != "rows":
            raise ValidationError("HostPipeline streams row chunks: it needs the row-major layout "
                                  "(a graph regrouped by tile_heavy serves device-resident passes only)")
        self.resident = bool(resident)
        self.device = device or g.device
        self.dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        # a row shard streams its own rows; labels and hot ranks cover all nodes
        self.n, self.n_nodes, self.k, self.s = g.n, g.n_nodes, k, g.s
        self.weighted = g.weighted
        dev = self.device
        off = g.offsets.cpu().numpy()
        self.bounds = plan_rows(off, max(1, chunks), k, self.weighted)
        self.arena = PinnedArena()
        pin = lambda t: None if t is None else self.arena.copy_of(t)  # noqa: E731
        # host copies of the prepared layout (the "stored graph")
        # the hot tier travels in compact form (bitmap, prefix, ranks)
        self.h_hot = None
        if g.hot_rank is not None and g.hot_bits is None:
            g.compact_hot()
        if g.hot_rank is not None and not self.resident:
            self.h_hot = [pin(g.hot_bits), pin(g.hot_pref), pin(g.hot_list)]
        self.n_hot = g.n_hot
        # packed targets (gee_pack_targets): per-8-arc-group bit-width deltas
        # and the real arcs' weights (pads rebuilt on the device)
        self.packed = (g.padded == 8 and not self.resident) if packed is None else bool(packed)
        if self.packed and (g.padded != 8 or self.resident):
            raise ValidationError("packed targets need rows padded to 8 arcs")
        self.sentinel = g.n_hot + g.n_nodes
        self.h_tgt = None if (self.packed or self.resident) else pin(g.targets)
        self.h_w = None if (self.packed or self.resident) else pin(g.weights)
        self.g = g if self.resident else None
        self.h_ctl, self.h_pay, self.h_wctl, self.h_wpay, self.wuni = [], [], [], [], []
        self.h_off = []
        self.views = []
        max_rows = max_arcs = 0
        for c in range(len(self.bounds) - 1):
            lo, hi = int(self.bounds[c]), int(self.bounds[c + 1])
            a0, a1 = int(off[lo]), int(off[hi])
            # chunk-relative offsets travel as int32 when the chunk allows it
            # (widened on the device): C4 saves 0.54 GB of H2D per call
            rel = off[lo:hi + 1] - off[lo]
            if rel[-1] < 2**31 and not self.resident:
                rel = rel.astype(np.int32)
            v = DeviceGraph(hi - lo, 0, dev)
            v.n_nodes = g.n_nodes
            if self.resident:  # the chunk's rebased offsets stay on the device
                v.res_off = torch.from_numpy(rel).to(dev)
                self.h_off.append(None)
            else:
                self.h_off.append(self.arena.copy_of(torch.from_numpy(rel)))
            # plan the chunk's heavy rows / block spans on a temporary device
            # copy of its rebased offsets (graph preparation)
            v.offsets = v.res_off if self.resident else self.h_off[c].to(dev).long()
            v.targets = torch.empty(a1 - a0, dtype=torch.int32, device=dev)  # shape only
            v.weights = None
            v._plan_heavy()
            ends = v.offsets[torch.arange(0, v.n + 32, 32, device=dev).clamp_(max=v.n)]
            v.max_block_arcs = int((ends[1:] - ends[:-1]).max().item()) if v.n else 0
            v.scale_exp, v.rel_err, v.max_row_abs = g.scale_exp, g.rel_err, g.max_row_abs
            v.hot_k, v.n_hot, v.hot_rank = k, g.n_hot, None
            v.padded = g.padded
            v.offsets = v.targets = None
            v.span = (lo, hi, a0, a1)
            if self.packed:
                self._pack_chunk(g, lo, hi, a0, a1)
            self.views.append(v)
            max_rows, max_arcs = max(max_rows, hi - lo), max(max_arcs, a1 - a0)
        # device slots (double-buffered) and the labels / hot ranks
        if self.packed:
            self.d_ctl = [torch.empty(max(1, max_arcs // 8), dtype=torch.uint8, device=dev) for _ in range(2)]
            # + 8 bytes: the bit reader loads the word after a value's last word
            self.d_pay = [torch.empty(max(t.numel() for t in self.h_pay) + 8, dtype=torch.uint8, device=dev)
                          for _ in range(2)]
            self.d_wctl = [torch.empty(max(1, max_arcs // 8), dtype=torch.uint8, device=dev)
                           if self.weighted else None for _ in range(2)]
            self.d_wpay = [torch.empty(max(1, max(t.numel() for t in self.h_wpay)), dtype=torch.uint8, device=dev)
                           if self.weighted else None for _ in range(2)]
            self.scratch_bytes = int(_lib.lib.gee_unpack_scratch_bytes(max_arcs // 8))
            self.d_scratch = torch.empty(max(1, self.scratch_bytes), dtype=torch.uint8, device=dev)
        slots = 0 if self.resident else 2
        self.d_off = [torch.empty(max_rows + 1, dtype=torch.int64, device=dev) for _ in range(slots)]
        self.d_off32 = [torch.empty(max_rows + 1, dtype=torch.int32, device=dev) for _ in range(slots)]
        self.d_tgt = [torch.empty(max_arcs, dtype=torch.int32, device=dev) for _ in range(slots)]
        self.d_w = [torch.empty(max_arcs, dtype=torch.float32, device=dev) if self.weighted else None
                    for _ in range(slots)]
        self.d_z = [torch.empty(max_rows * k, dtype=torch.float32, device=dev) for _ in range(2)]
        self.d_y = torch.empty(self.n_nodes, dtype=torch.int32, device=dev)
        self.d_hot = [torch.empty_like(t, device=dev) for t in self.h_hot] if self.h_hot is not None else None
        self.proj = DeviceGraph(self.n_nodes, 0, dev)  # what project() needs: the hot tier of all nodes
        if self.d_hot is not None:
            self.proj.hot_bits, self.proj.hot_pref, self.proj.hot_list = self.d_hot
            self.proj.n_hot = self.n_hot
        elif self.resident and g.hot_rank is not None:
            self.proj.hot_bits, self.proj.hot_pref, self.proj.hot_list = g.hot_bits, g.hot_pref, g.hot_list
            self.proj.n_hot = self.n_hot
        self.s_in = torch.cuda.Stream(dev)
        self.s_cmp = torch.cuda.Stream(dev)
        self.s_out = torch.cuda.Stream(dev)

    def _pack_chunk(self, g, lo, hi, a0, a1):
        """Graph preparation: code chunk [lo, hi)'s padded targets and weights
        (device) and keep the packed streams in pinned memory."""
        dev = g.device
        groups = (a1 - a0) // 8
        off = g.offsets[lo:hi + 1] - g.offsets[lo]
        tgt = g.targets[a0:a1]
        wts = g.weights[a0:a1] if self.weighted else None
        u8 = lambda m: torch.empty(max(1, m), dtype=torch.uint8, device=dev)  # noqa: E731
        ctl, pay = u8(groups), u8(4 * (a1 - a0))
        wctl, wpay = (u8(groups), u8(4 * (a1 - a0))) if self.weighted else (None, None)
        nb, nwb = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.lib.gee_pack_targets(_lib.ptr(off), hi - lo, _lib.ptr(tgt), _lib.ptr(wts), a1 - a0,
                                             self.sentinel, _lib.ptr(ctl), _lib.ptr(pay), ctypes.byref(nb),
                                             _lib.ptr(wctl), _lib.ptr(wpay), ctypes.byref(nwb),
                                             _lib.stream_handle()), "gee_pack_targets")
        pin = self.arena.copy_of
        self.h_ctl.append(pin(ctl[:groups]))
        self.h_pay.append(pin(pay[:int(nb.value)]))
        empty = torch.empty(0, dtype=torch.uint8)
        # one weight code for the whole chunk (C4: every group is 3-byte fixed
        # point with e = 24): send it instead of the per-group bytes
        wu = -1
        if self.weighted and groups:
            w0 = int(wctl[0])
            if bool((wctl[:groups] == w0).all()):
                wu = w0
        self.wuni.append(wu)
        self.h_wctl.append(pin(wctl[:groups]) if self.weighted and wu < 0 else empty)
        self.h_wpay.append(pin(wpay[:int(nwb.value)]) if self.weighted else empty)
        del pay, wpay

    @property
    def n_chunks(self):
        return len(self.views)

    def h2d_bytes(self, h_labels):
        b = h_labels.numel() * h_labels.element_size()
        if self.resident:
            return int(b)
        b += sum(t.numel() * t.element_size() for t in self.h_off)
        if self.packed:
            b += sum(t.numel() for t in self.h_ctl) + sum(t.numel() for t in self.h_pay)
            b += sum(t.numel() for t in self.h_wctl) + sum(t.numel() for t in self.h_wpay)
        else:
            b += self.h_tgt.numel() * 4
            if self.h_w is not None:
                b += self.h_w.numel() * 4
        if self.h_hot is not None:
            b += sum(t.numel() * 4 for t in self.h_hot)
        return int(b)

    def _sparse_slots(self):
        if getattr(self, "cm", None) is not None:
            return
        dev, k = self.device, self.k
        rows = max(hi - lo for lo, hi, _, _ in (v.span for v in self.views)) if self.views else 0
        mw = (k + 63) // 64
        nb = int(_lib.lib.gee_zc_blocks(rows))
        self.cm = [torch.empty(rows * mw, dtype=torch.int64, device=dev) for _ in range(2)]
        self.cb = [torch.empty(nb + 1, dtype=torch.int64, device=dev) for _ in range(2)]
        self.cv = [torch.empty(rows * k, dtype=torch.float32, device=dev) for _ in range(2)]
        hs = self.HOST_SLOTS
        self.hm = [self.arena.empty(rows * mw, torch.int64) for _ in range(hs)]
        self.hb = [self.arena.empty(nb + 1, torch.int64) for _ in range(hs)]
        self.hv = [self.arena.empty(rows * k, torch.float32) for _ in range(hs)]
        self.h_tot = self.arena.empty(max(1, len(self.views)), torch.int64).zero_()
        self.mw = mw

    def run(self, h_labels, h_z, emb: Embedder, sparse=True, inv=None, dense_every=None):
        """labels (pinned host int32[n]) -> h_z (pinned host float32[n, k]).
        ``inv`` (float64[k+1]) replaces 1/count (a caller's projection).
        With ``sparse``, every ``dense_every``-th chunk still leaves dense,
        copied by the DMA engine straight into h_z: the host threads that
        rebuild the row-sparse chunks are the bound once the graph does not
        cross PCIe (resident), and the device-to-host direction is otherwise
        idle (default: every 8th chunk when resident, none when streaming,
        where the copy-in is the bound)."""
        if h_z.shape != (self.n, self.k) or h_z.dtype != torch.float32 or not h_z.is_contiguous():
            raise ValidationError("h_z must be a contiguous float32 (n, k) host tensor")
        if sparse:
            self._sparse_slots()
        if dense_every is None:
            dense_every = self.DENSE_EVERY_RESIDENT if self.resident else self.DENSE_EVERY_STREAMED
        nv = len(self.views)
        self._dense = [(not sparse) or (dense_every > 0 and i % dense_every == dense_every - 1) for i in range(nv)]
        self._last_compact = [-1, -1]  # last sparse chunk that used each device compaction slot
        ev = lambda: torch.cuda.Event()  # noqa: E731
        e_lab = ev()
        with torch.cuda.stream(self.s_in):
            self.d_y.copy_(h_labels, non_blocking=True)
            if self.d_hot is not None:
                for d, h in zip(self.d_hot, self.h_hot):
                    d.copy_(h, non_blocking=True)
            e_lab.record(self.s_in)
        self.s_cmp.wait_event(e_lab)
        with torch.cuda.stream(self.s_cmp):
            emb.project(self.d_y, validate=False, g=self.proj, inv=inv)
        nv = len(self.views)
        e_in = [ev() for _ in self.views]
        self._copyin_done = e_in[-1] if e_in else None
        self._last_issued = False  # (an event not yet recorded queries as complete)
        e_cmp = [ev() for _ in self.views]
        e_out = [ev() for _ in self.views]
        self.d2h_bytes = 0
        # sparse copy-out: a host worker drains chunk i (its size is known once
        # the chunk is compacted) and expands chunk i-1 into h_z, so the main
        # thread keeps the copy-in and compute queues fed meanwhile
        recorded = [threading.Event() for _ in self.views]
        drained = [threading.Event() for _ in self.views]
        errors = []
        worker = None
        if sparse and nv:
            worker = threading.Thread(target=self._sparse_worker,
                                      args=(e_cmp, e_out, h_z, recorded, drained, errors), daemon=True)
            worker.start()
        try:
            for i, v in enumerate(self.views):
                self._issue_chunk(i, v, emb, h_z, sparse, e_in, e_cmp, e_out, drained, errors)
                self._last_issued = i == nv - 1
                recorded[i].set()
        except BaseException as e:
            errors.append(e)  # stops the worker before it drains an unissued chunk
            raise
        finally:
            for r in recorded:
                r.set()  # a failed issue must not leave the worker waiting
            if worker is not None:
                worker.join()
        if errors:
            raise errors[0]
        self.s_out.synchronize()
        for v in self.views:
            v.offsets = v.targets = v.weights = None
        return h_z

    def _issue_chunk(self, i, v, emb, h_z, sparse, e_in, e_cmp, e_out, drained, errors):
        """Main thread: queue chunk i's copy-in, decode, pull and compaction
        (resident: the pull on the HBM-resident rows and the compaction)."""
        b = i & 1
        lo, hi, a0, a1 = v.span
        with torch.cuda.stream(self.s_in):
            if not self.resident:
                if i >= 2:
                    self.s_in.wait_event(e_cmp[i - 2])  # slot b's CSR is free
                ho = self.h_off[i]
                (self.d_off32 if ho.dtype == torch.int32 else self.d_off)[b][:hi - lo + 1].copy_(ho, non_blocking=True)
                if self.packed:
                    self.d_ctl[b][:self.h_ctl[i].numel()].copy_(self.h_ctl[i], non_blocking=True)
                    self.d_pay[b][:self.h_pay[i].numel()].copy_(self.h_pay[i], non_blocking=True)
                    if self.weighted:
                        if self.h_wctl[i].numel():
                            self.d_wctl[b][:self.h_wctl[i].numel()].copy_(self.h_wctl[i], non_blocking=True)
                        self.d_wpay[b][:self.h_wpay[i].numel()].copy_(self.h_wpay[i], non_blocking=True)
                else:
                    self.d_tgt[b][:a1 - a0].copy_(self.h_tgt[a0:a1], non_blocking=True)
                    if self.weighted:
                        self.d_w[b][:a1 - a0].copy_(self.h_w[a0:a1], non_blocking=True)
            e_in[i].record(self.s_in)
        self.s_cmp.wait_event(e_in[i])
        dense = self._dense[i]
        if i >= 2 and self._dense[i - 2]:
            self.s_cmp.wait_event(e_out[i - 2])  # Z slot b has been copied out
        with torch.cuda.stream(self.s_cmp):
            if self.resident:
                v.offsets = v.res_off
                v.targets = self.g.targets[a0:a1]
                v.weights = self.g.weights[a0:a1] if self.weighted else None
            else:
                if self.h_off[i].dtype == torch.int32:  # widen on the device
                    _lib.check(_lib.lib.gee_widen_offsets(_lib.ptr(self.d_off32[b]), hi - lo + 1,
                                                          _lib.ptr(self.d_off[b]), _lib.stream_handle(self.s_cmp)),
                               "gee_widen_offsets")
                if self.packed:  # (the decoder marks row starts from the offsets)
                    wu = self.wuni[i]
                    _lib.check(_lib.lib.gee_unpack_targets(
                        _lib.ptr(self.d_ctl[b]), _lib.ptr(self.d_pay[b]), (a1 - a0) // 8, _lib.ptr(self.d_off[b]),
                        hi - lo, _lib.ptr(self.d_wctl[b]) if self.weighted and wu < 0 else None, wu,
                        _lib.ptr(self.d_wpay[b]) if self.weighted else None, self.sentinel, _lib.ptr(self.d_tgt[b]),
                        _lib.ptr(self.d_w[b]) if self.weighted else None, _lib.ptr(self.d_scratch),
                        self.scratch_bytes, _lib.stream_handle(self.s_cmp)), "gee_unpack_targets")
                v.offsets = self.d_off[b][:hi - lo + 1]
                v.targets = self.d_tgt[b][:a1 - a0]
                v.weights = self.d_w[b][:a1 - a0] if self.weighted else None
            z = self.d_z[b][:(hi - lo) * self.k].view(hi - lo, self.k)
            emb.pull(v, z)
            if not dense:
                j = self._last_compact[b]  # the previous sparse chunk on compaction slot b
                if j >= 0:
                    drained[j].wait()  # the worker has queued chunk j's copy-out
                    if errors:
                        raise errors[0]
                    self.s_cmp.wait_event(e_out[j])  # compact slot b has been copied out
                self._last_compact[b] = i
                _lib.check(_lib.lib.gee_z_compact(_lib.ptr(z), hi - lo, self.k, _lib.ptr(self.cm[b]),
                                                  _lib.ptr(self.cb[b]), _lib.ptr(self.cv[b]),
                                                  _lib.stream_handle(self.s_cmp)), "gee_z_compact")
                nb = int(_lib.lib.gee_zc_blocks(hi - lo))
                self.h_tot[i:i + 1].copy_(self.cb[b][nb:nb + 1], non_blocking=True)
            e_cmp[i].record(self.s_cmp)
        if dense:
            self.s_out.wait_event(e_cmp[i])
            with torch.cuda.stream(self.s_out):
                h_z[lo:hi].copy_(z, non_blocking=True)
                e_out[i].record(self.s_out)
            self.d2h_bytes += z.numel() * 4

    def _sparse_worker(self, e_cmp, e_out, h_z, recorded, drained, errors):
        """Host workers: a drainer queues chunk i's row-sparse copy-out as
        soon as the chunk is compacted, and an expander rebuilds each copied
        chunk's dense rows in h_z; HOST_SLOTS host slots let the next copies
        proceed while a chunk expands (drain(i) reuses the slot of chunk
        i - HOST_SLOTS once that one is expanded)."""
        nv = len(self.views)
        expanded = [threading.Event() for _ in range(nv)]

        def expander():
            try:
                torch.cuda.set_device(self.dev_index)
                for i in range(nv):
                    drained[i].wait()
                    if errors:
                        return
                    if not self._dense[i]:  # a dense chunk went straight into h_z
                        self._expand(i, e_out, h_z)
                    expanded[i].set()
            except BaseException as e:  # surfaced by run()
                errors.append(e)
            finally:
                for x in expanded:
                    x.set()

        ex = threading.Thread(target=expander, daemon=True)
        ex.start()
        try:
            torch.cuda.set_device(self.dev_index)
            for i in range(nv):
                recorded[i].wait()
                if errors:
                    return
                if not self._dense[i]:
                    if i >= self.HOST_SLOTS:
                        expanded[i - self.HOST_SLOTS].wait()
                        if errors:
                            return
                    self._drain(i, e_cmp, e_out)
                drained[i].set()
        except BaseException as e:  # surfaced by run()
            errors.append(e)
        finally:
            for d in drained:
                d.set()
            ex.join()

    def _drain(self, i, e_cmp, e_out):
        """Host: once chunk i is compacted, copy its sparse Z out (size now known)."""
        lo, hi, _, _ = self.views[i].span
        b = i & 1  # device compaction slot
        h = i % self.HOST_SLOTS  # host slot
        e_cmp[i].synchronize()
        tot = int(self.h_tot[i])
        rows = hi - lo
        nb = int(_lib.lib.gee_zc_blocks(rows))
        with torch.cuda.stream(self.s_out):
            self.hm[h][:rows * self.mw].copy_(self.cm[b][:rows * self.mw], non_blocking=True)
            self.hb[h][:nb + 1].copy_(self.cb[b][:nb + 1], non_blocking=True)
            if tot:
                self.hv[h][:tot].copy_(self.cv[b][:tot], non_blocking=True)
            e_out[i].record(self.s_out)
        self.d2h_bytes += 8 * (rows * self.mw + nb + 1) + 4 * tot

    def _expand_threads(self):
        if self.EXPAND_THREADS is not None:
            return int(self.EXPAND_THREADS)
        if self.resident:
            return self.EXPAND_THREADS_RESIDENT
        # once the last chunk's copy-in has landed, the DMA reads are done:
        # the tail chunks expand on every host thread
        done = self._copyin_done
        if self._last_issued and done is not None and done.query():
            return 0
        return self.EXPAND_THREADS_STREAMED

    def _expand(self, i, e_out, h_z):
        """Host: rebuild chunk i's dense Z rows in the caller's buffer."""
        from .formats import io_lib

        lo, hi, _, _ = self.views[i].span
        h = i % self.HOST_SLOTS
        e_out[i].synchronize()
        rc = io_lib().gee_io_expand_rows(_lib.ptr(self.hm[h]), _lib.ptr(self.hv[h]), _lib.ptr(self.hb[h]), hi - lo,
                                         self.k, ctypes.c_void_p(h_z.data_ptr() + lo * self.k * 4),
                                         self._expand_threads())
        if rc:
            raise ValidationError(io_lib().gee_io_last_error().decode())


def pinned_like(shape, dtype=torch.float32):
    return torch.empty(shape, dtype=dtype).pin_memory()


__all__ = ["HostPipeline", "PinnedArena", "pinned_like", "np"]
