"""HBM-resident graphs and the edge-pass engine over the C ABI.

torch provides device memory and streams only; every byte of the edge pass
is computed by libgee_b200.so (include/gee_b200.h).  Nothing here falls back
to the CPU: without a CUDA device the calls raise.
"""

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr
from .errors import ValidationError


def require_cuda(device=None):
    if not torch.cuda.is_available():
        raise _lib.CudaError("the GEE edge pass runs on a CUDA device (sm_100a); none is visible")
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def to_device(a, dtype, device):
    """numpy / torch array -> contiguous CUDA tensor of `dtype`."""
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype).contiguous()
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.to(device=device, dtype=dtype, non_blocking=False).contiguous()


def _stream():
    return _lib.stream_handle()


class DeviceGraph:
    """A listed edge multiset resident in HBM, laid out for the edge pass.

    pull layout  symmetric CSR: row x holds (v, w) for every listed edge
                 touching x (both endpoints; self-loops twice) -- the
                 reference's SOURCE_ONLY storage (encoder.py:37-55) -- plus
                 the tile plan (tile_row) and the fixed-point exponent.
    push layout  the COO lists themselves (src, dst, w) with the edge rule
                 (both updates, or source-only for arc lists).
    """

    def __init__(self, n, s_listed, device):
        self.n = int(n)  # rows of this layout (a shard's local rows)
        self.n_nodes = int(n)  # nodes the labels cover (global for a shard)
        self.s = int(s_listed)  # listed edges: the GEPS numerator
        self.device = device
        self.offsets = self.targets = self.weights = None
        # rows heavier than HEAVY_ARCS: the heavy-item reducer (k <= 255) or
        # the wide kernel's CTA-per-row path (k > 255)
        self.heavy_rows = None
        self.n_heavy = 0
        self.short_rows = None
        self.short_arcs = 0
        self.max_block_arcs = 0
        self.scale_exp = 0
        self.rel_err = 0.0
        self.max_row_abs = self.max_abs = self.min_abs = 0.0
        self.src = self.dst = self.w = None
        self.coo_source_only = False
        self.hot_rank = None  # int32[n_nodes]: degree rank of hot vertices, -1 cold
        # the same tier in compact form for the per-call projection (compact_hot)
        self.hot_bits = self.hot_pref = self.hot_list = None
        self.global_offsets = None  # row shard: global symmetric offsets until the hot plan
        self.n_hot = 0
        self.hot_k = None  # k the hot tier was planned for (None = not planned)
        self._owns_targets = False
        self._owns_weights = False
        self.padded = 0  # rows padded to a multiple of this many arcs (0: not padded)
        # "rows": heavy rows inside the row-major CSR; "tiles": relocated into
        # the tile-major region behind the light rows (tile_heavy)
        self.heavy_layout = "rows"
        self.n_tiles = 0
        self.l2_arcs = self.light_arcs = 0
        self.group_dst = None
        self.arcs_unpadded = None

    # ---------------------------------------------------------------- build
    @classmethod
    def from_edges(cls, src, dst, w, n, device=None, pull=True, keep_coo=False, stable=False):
        """Upload a listed edge list and build the requested layouts."""
        dev = require_cuda(device)
        g = cls(n, len(src), dev)
        src_d = to_device(src, torch.int32, dev)
        dst_d = to_device(dst, torch.int32, dev)
        w_d = to_device(w, torch.float32, dev)
        if pull:
            g._build_sym(src_d, dst_d, w_d, stable)
        if keep_coo or not pull:
            g.src, g.dst, g.w = src_d, dst_d, w_d
        return g

    @classmethod
    def from_csr(cls, offsets, targets, weights, n, symmetric, device=None, pull=True, keep_coo=False):
        """Upload a stored CsrGraph.

        symmetric=True  (SOURCE_ONLY storage: each listed undirected edge is
                         two arcs) -> already the pull layout; listed edges =
                         arcs / 2.
        symmetric=False (BOTH_ENDPOINTS storage: one arc per listed edge)
                         -> expanded to COO and mirrored for pull.
        """
        dev = require_cuda(device)
        off_d = to_device(offsets, torch.int64, dev)
        tgt_d = to_device(targets, torch.int32, dev)
        w_d = to_device(weights, torch.float32, dev)
        arcs = int(tgt_d.numel())
        if symmetric:
            g = cls(n, arcs // 2, dev)
            g.offsets, g.targets, g.weights = off_d, tgt_d, w_d
            g._owns_targets = not (isinstance(targets, torch.Tensor) and targets.data_ptr() == tgt_d.data_ptr())
            g._owns_weights = w_d is not None and not (isinstance(weights, torch.Tensor) and
                                                       weights.data_ptr() == w_d.data_ptr())
            g._plan()
            if keep_coo or not pull:
                rows = torch.empty(arcs, dtype=torch.int32, device=dev)
                check(lib.gee_csr_rows(ptr(off_d), n, arcs, ptr(rows), _stream()), "gee_csr_rows")
                g.src, g.dst, g.w, g.coo_source_only = rows, tgt_d, w_d, True
            return g
        g = cls(n, arcs, dev)
        rows = torch.empty(arcs, dtype=torch.int32, device=dev)
        if arcs:
            check(lib.gee_csr_rows(ptr(off_d), n, arcs, ptr(rows), _stream()), "gee_csr_rows")
        if pull:
            g._build_sym(rows, tgt_d, w_d, stable=False)
        if keep_coo or not pull:
            g.src, g.dst, g.w = rows, tgt_d, w_d
        return g

    def to_source_only_coo(self):
        """Expose the symmetric (pull) CSR as a SOURCE_ONLY arc list for the
        push: src = row of each arc, dst = its target.  Only before the hot
        tier rewrites the targets into label-table slots."""
        if self.hot_k is not None and self.hot_rank is not None:
            raise ValidationError("the hot tier already rewrote the targets; build the push layout first")
        arcs = int(self.targets.numel())
        rows = torch.empty(arcs, dtype=torch.int32, device=self.device)
        if arcs:
            check(lib.gee_csr_rows(ptr(self.offsets), self.n, arcs, ptr(rows), _stream()), "gee_csr_rows")
        self.src, self.dst, self.w, self.coo_source_only = rows, self.targets, self.weights, True
        return self

    def _build_sym(self, src_d, dst_d, w_d, stable):
        n, s, dev = self.n, int(src_d.numel()), self.device
        self.offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
        self.targets = torch.empty(2 * s, dtype=torch.int32, device=dev)
        self.weights = torch.empty(2 * s, dtype=torch.float32, device=dev) if w_d is not None else None
        check(lib.gee_build_csr(ptr(src_d), ptr(dst_d), ptr(w_d), s, n, 1, 1 if stable else 0,
                                ptr(self.offsets), ptr(self.targets), ptr(self.weights), _stream()),
              "gee_build_csr")
        self._owns_targets = True
        self._owns_weights = True
        self._plan()

    def _plan(self):
        """Pull planning (graph preparation): weight statistics + fixed-point
        exponent, heavy-row work items, block arc spans."""
        arcs = self.arcs
        self._plan_heavy()
        mx, mn, mxa = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        nf = ctypes.c_int32()
        check(lib.gee_graph_stats(ptr(self.offsets), ptr(self.weights), self.n, arcs, ctypes.byref(mx),
                                  ctypes.byref(mn), ctypes.byref(mxa), ctypes.byref(nf), _stream()),
              "gee_graph_stats")
        if nf.value:
            raise ValidationError("arc weights must be finite")
        self.max_row_abs, self.max_abs, self.min_abs = mx.value, mxa.value, mn.value
        self._set_scale(mx.value, mxa.value, mn.value)
        # arc span of the widest 32-row block (gee_reduce_blocks keeps
        # block-local offsets in int32)
        ends = self.offsets[torch.arange(0, self.n + 32, 32, device=self.device).clamp_(max=self.n)]
        self.max_block_arcs = int((ends[1:] - ends[:-1]).max().item()) if self.n else 0

    HEAVY_ARCS = 2048  # rows above go to the heavy path (<= the block reducer's limit)
    HEAVY_ITEM_ARCS = 65536  # arcs per heavy work item (one warp)

    def _set_scale(self, max_row_abs, max_abs, min_abs):
        e, rel = ctypes.c_int32(), ctypes.c_double()
        check(lib.gee_block_scale_exp(max_row_abs, max_abs, min_abs, ctypes.byref(e), ctypes.byref(rel)),
              "gee_block_scale_exp")
        self.scale_exp, self.rel_err = e.value, rel.value

    def weight_stats(self):
        """(max row |w| sum, max |w|, min nonzero |w|) of this layout's arcs."""
        return self.max_row_abs, self.max_abs, self.min_abs

    def adopt_scale(self, stats):
        """Use the fixed-point exponent of the whole graph this layout is a row
        shard of.  `stats` = (max over shards of max_row_abs and max_abs, min
        over shards of the nonzero min_abs); the exponent it gives is <= this
        shard's own, so no sum can overflow, and every shard then rounds
        each weight exactly as the single-GPU pull does (bit-identical rows)."""
        mx, mxa, mn = (float(v) for v in stats)
        self._set_scale(mx, mxa, mn)

    def _plan_heavy(self):
        """Heavy-row work items (graph preparation)."""
        n = self.n
        rows = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        nh = ctypes.c_int64()
        check(lib.gee_reduce_heavy_plan(ptr(self.offsets), n, self.HEAVY_ARCS, ptr(rows), ctypes.byref(nh),
                                        _stream()), "gee_reduce_heavy_plan")
        self.n_heavy = int(nh.value)
        self.heavy_arc_total = 0
        self.item_first = self.item_end = self.item_row = self.item_slot = self.mega_rows = None
        self.n_items = self.n_mega = 0
        if self.n_heavy == 0:
            self.heavy_rows = None
            return
        # ascending row order: the chunk pass then streams the CSR and the
        # finalize sweeps Z in address order (k_mark_heavy appends in
        # atomic order, which scatters both over 30 GB)
        rows = torch.sort(rows[:self.n_heavy])[0].contiguous()
        r64 = rows.to(torch.int64)
        first = self.offsets[r64].cpu()
        deg = (self.offsets[r64 + 1] - self.offsets[r64]).cpu()
        self.heavy_arc_total = int(deg.sum())
        self._make_items(rows, first, deg)

    def _make_items(self, rows, first, deg):
        """Work items of gee_reduce_heavy for the heavy `rows` (device int32,
        ascending) whose arcs are cls / weights [first, first + deg) (host
        int64)."""
        # work items of gee_reduce_heavy: runs of <= HEAVY_ITEM_ARCS arcs;
        # rows with several items ("mega" rows) combine through acc + finalize
        nit = (deg + self.HEAVY_ITEM_ARCS - 1) // self.HEAVY_ITEM_ARCS
        it_row = torch.repeat_interleave(torch.arange(self.n_heavy), nit)
        it_j = torch.arange(int(nit.sum())) - torch.repeat_interleave(torch.cumsum(nit, 0) - nit, nit)
        it_first = first[it_row] + it_j * self.HEAVY_ITEM_ARCS
        it_end = torch.minimum(it_first + self.HEAVY_ITEM_ARCS, first[it_row] + deg[it_row])
        mega = nit > 1
        mega_idx = torch.full((self.n_heavy,), -1, dtype=torch.int64)
        mega_idx[mega] = torch.arange(int(mega.sum()))
        rows_cpu = rows.cpu()
        # largest items first (the kernel fetches them dynamically)
        order = torch.argsort(it_end - it_first, descending=True, stable=True)
        it_row, it_first, it_end = it_row[order], it_first[order], it_end[order]
        self.item_first = it_first.to(self.device)
        self.item_end = it_end.to(self.device)
        self.item_row = rows_cpu[it_row].to(torch.int32).to(self.device)
        self.item_slot = mega_idx[it_row].to(torch.int32).to(self.device)
        self.n_items = int(it_row.numel())
        self.mega_rows = rows_cpu[mega].to(torch.int32).to(self.device)
        self.n_mega = int(mega.sum())
        self.heavy_rows = rows

    # Hot-label tier (csrc/gee_hot.cu): worth it when the packed label array
    # outgrows what L2 keeps resident under random access and degrees are
    # skewed (R-MAT); ER graphs end up with few or no hot vertices.
    HOT_MIN_TABLE_BYTES = 16 << 20
    # the top 16M vertices by degree: with rows sorted by slot, ranking more
    # (up to all 60M with an arc) trims the lookups' DRAM reads but the
    # histogram's rank scatter grows more (C4 step: 16M 21.32 ms, 32M 21.39,
    # 64M 21.53)
    HOT_MAX = 16 << 20
    HOT_MIN_DEGREE = 1

    def prepare_hot(self, k, enable=None):
        """Plan the hot tier for k classes (once; rewrites the pull targets)."""
        if self.hot_k == k or not self.has_pull:
            return
        if self.hot_k is not None:
            raise ValidationError("hot tier already planned for a different k")
        table_bytes = int(lib.gee_label_table_bytes(self.n_nodes, 0, k))
        # a row shard ranks the GLOBAL vertices by their global degree
        deg_off = self.offsets if self.n == self.n_nodes else self.global_offsets
        if enable is None:
            enable = table_bytes > self.HOT_MIN_TABLE_BYTES and k <= 65535 and deg_off is not None
        self.hot_k = k
        if not enable or self.arcs == 0 or deg_off is None:
            self.global_offsets = None
            self._sort_rows()
            self._pad_rows()
            return
        self._own_pull_arrays()
        n = self.n_nodes
        self.hot_rank = torch.empty(n, dtype=torch.int32, device=self.device)
        nh = ctypes.c_int64()
        # slots are int32: every slot n_hot + v, and the sentinel n_hot + n,
        # must stay below 2^31
        max_hot = min(n, self.HOT_MAX // int(lib.gee_label_bytes(k)), 2**31 - 1 - n - 1)
        if max_hot <= 0:
            self.hot_rank = None
            self._sort_rows()
            self._pad_rows()
            return
        check(lib.gee_hot_plan(ptr(deg_off), n, max_hot, self.HOT_MIN_DEGREE, ptr(self.hot_rank), None, ctypes.byref(nh),
                               _stream()), "gee_hot_plan")
        self.global_offsets = None
        self.n_hot = int(nh.value)
        if self.n_hot == 0:
            self.hot_rank = None
            return
        check(lib.gee_hot_encode(ptr(self.targets), self.arcs, ptr(self.hot_rank), self.n_hot, _stream()),
              "gee_hot_encode")
        self.compact_hot()
        self._sort_rows()
        self._pad_rows()

    def compact_hot(self):
        """hot_rank (int32 per vertex) -> hot_bits (u32 bitmap of the hot
        vertices), hot_pref (hot vertices before each word) and hot_list (their
        ranks in vertex order): what gee_build_projection_hotc reads each call
        (graph preparation)."""
        hr = self.hot_rank
        n = hr.numel()
        nw = (n + 31) // 32
        hot = torch.zeros(nw * 32, dtype=torch.bool, device=hr.device)
        hot[:n] = hr >= 0
        hv = hot.view(nw, 32).to(torch.int64)
        bits = (hv << torch.arange(32, device=hr.device, dtype=torch.int64)).sum(1)
        self.hot_bits = torch.where(bits >= 2**31, bits - 2**32, bits).to(torch.int32)  # u32 bit pattern
        cnt = hv.sum(1)
        self.hot_pref = (torch.cumsum(cnt, 0) - cnt).to(torch.int32)
        self.hot_list = hr[hot[:n]].contiguous()
        del hv, bits, cnt, hot

    PAD_ROWS = 8  # every row padded to a multiple of 8 arcs (the block reducer's lane unit)
    # rows this short skip the weighted block reducer's windows (0: off; <= 4).
    # C4 block reducer: 0 / 1 / 2 / 3 / 4 -> 7.49 / 7.23 / 7.17 / 7.21 / 7.29 ms
    SHORT_ROW_ARCS = 2

    def _pad_rows(self):
        """Pad each row's arc run to a multiple of PAD_ROWS with (sentinel
        slot, weight 0) arcs (graph preparation): every lane of the block
        reducer then owns arcs of one row.  The sentinel slot's label is 0."""
        align = self.PAD_ROWS
        if self.arcs == 0 or self.padded:
            return
        poff = torch.empty(self.n + 1, dtype=torch.int64, device=self.device)
        pa = ctypes.c_int64()
        check(lib.gee_pad_offsets(ptr(self.offsets), self.n, align, ptr(poff), ctypes.byref(pa), _stream()),
              "gee_pad_offsets")
        pa = int(pa.value)
        tgt = torch.empty(pa, dtype=torch.int32, device=self.device)
        wts = torch.empty(pa, dtype=torch.float32, device=self.device) if self.weights is not None else None
        sentinel = self.n_hot + self.n_nodes
        check(lib.gee_pad_rows(ptr(self.offsets), ptr(poff), self.n, ptr(self.targets), ptr(self.weights), sentinel,
                               ptr(tgt), ptr(wts), _stream()), "gee_pad_rows")
        self.arcs_unpadded = self.arcs
        # rows of 1 .. SHORT_ROW_ARCS arcs, one bit per row (uint32 per 32-row
        # block): the weighted block reducer stores their Z entries directly
        nb = (self.n + 31) // 32
        bits = torch.zeros(nb * 32, dtype=torch.int64, device=self.device)
        deg = self.offsets[1:] - self.offsets[:-1]
        bits[:self.n] = (deg >= 1) & (deg <= self.SHORT_ROW_ARCS)
        one = (bits.view(nb, 32) << torch.arange(32, device=self.device)).sum(1)
        self.short_rows = torch.where(one >= 2**31, one - 2**32, one).to(torch.int32).contiguous()
        self.short_arcs = self.SHORT_ROW_ARCS
        del deg
        del bits, one
        self.offsets, self.targets, self.weights = poff, tgt, wts
        self._owns_targets = self._owns_weights = True
        self.padded = align
        self._plan()

    # Tile-major heavy region (csrc/gee_tiles.cu).  A tile is a run of
    # label-table slots that fits one CTA's shared memory as bytes; slots past
    # TILE_MAX tiles stay on the L2 lookup path (the region's tail segment).
    # C4 step by tile count (192 KB tiles): 8: 18.5 ms, 21: 18.3, 42: 18.5,
    # 86 (the whole hot tier): 19.5 -- the sparse upper tiles hold spans of a
    # few arcs, whose scattered class writes cost more than their L2 lookups
    # (224 KB tiles: slower, the streams need some L1).
    TILE_SLOTS = 196608
    TILE_MAX = 21
    # arcs each (tile, row) span is padded to (a multiple of 16, the scatter's group): 32 makes every span's
    # class bytes whole 32-byte sectors.  C4 tail + tiles / heavy reducer / step: 16: 3.17 / 2.24 / 17.53 ms,
    # 32: 3.03 / 2.28 / 17.38 ms, 64: 3.26 / 2.48 / 17.81 ms
    SPAN_ALIGN = 32

    def tile_heavy(self, tile_slots=None, max_tiles=None):
        """Regroup the heavy rows' targets by slot tile (graph preparation;
        after prepare_hot).  The arrays become
            targets  [ light rows, row-major | heavy tail | tile 0 | tile 1 | ... ]
            weights  [ light rows, row-major | heavy rows, row-major (row, tile, slot) ]
        (the class stream is indexed like the weights), every (tile, row)
        span padded to SPAN_ALIGN arcs in both orders, and group_dst maps the 16-arc
        groups of the heavy targets to their place in the row-major order.
        Heavy rows keep an empty run in `offsets` (the block reducer
        zero-fills them, gee_reduce_heavy then writes them).  Returns True
        when the layout changed."""
        if self.heavy_layout == "tiles" or not self.padded or self.n_heavy == 0 or self.hot_k is None:
            return False
        if self.hot_k > 255:
            return False
        ts = int(tile_slots or self.TILE_SLOTS)
        mt = int(max_tiles or self.TILE_MAX)
        if ts % 16 or ts < 16:
            raise ValidationError("tile_slots must be a multiple of 16")
        dev, n, H = self.device, self.n, self.n_heavy
        sentinel = self.n_hot + self.n_nodes
        T = min(mt, (sentinel + ts - 1) // ts)
        if T <= 0:
            return False
        st = _stream()
        thr = torch.tensor([s * ts for s in range(T)] + [min(T * ts, sentinel), sentinel], dtype=torch.int64,
                           device=dev)
        bounds = torch.empty((T + 2) * H, dtype=torch.int64, device=dev)
        check(lib.gee_tile_bounds(ptr(self.offsets), ptr(self.heavy_rows), H, ptr(self.targets), ptr(thr), T + 2,
                                  ptr(bounds), st), "gee_tile_bounds")
        bounds = bounds.view(T + 2, H)
        seg_len = bounds[1:] - bounds[:-1]  # (T + 1, H): tiles 0..T-1, then the tail; row padding dropped
        al = int(self.SPAN_ALIGN)
        if al < 16 or al % 16:
            raise ValidationError("SPAN_ALIGN must be a multiple of 16")
        seg_pad = (seg_len + al - 1) // al * al
        # light rows, compacted
        lens = self.offsets[1:] - self.offsets[:-1]
        lens[self.heavy_rows.to(torch.int64)] = 0
        poff = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        torch.cumsum(lens, 0, out=poff[1:])
        light = int(poff[-1].item())
        light16 = (light + 31) // 32 * 32
        total = int(light16 + seg_pad.sum().item())
        # tile-major order of the targets: tail first, then the tiles
        order = [T] + list(range(T))
        src_first = bounds[:-1][order].reshape(-1).contiguous()
        src_len = seg_len[order].reshape(-1).contiguous()
        dst_len = seg_pad[order].reshape(-1).contiguous()
        t_first = torch.cumsum(dst_len, 0) - dst_len + light16  # (T + 1, H) flattened, region order
        # row-major order of the weights / class stream: (row, tile 0..T-1, tail)
        rp = seg_pad.t().contiguous()  # (H, T + 1)
        r_first = (torch.cumsum(rp.reshape(-1), 0) - rp.reshape(-1) + light16).view(H, T + 1)
        r_first_o = r_first.t()[order].reshape(-1).contiguous()  # same span order as t_first
        tgt = torch.empty(total, dtype=torch.int32, device=dev)
        wts = torch.empty(total, dtype=torch.float32, device=dev) if self.weights is not None else None
        if light16 > light:
            tgt[light:light16] = sentinel
            if wts is not None:
                wts[light:light16] = 0
        check(lib.gee_span_copy(n, ptr(self.offsets), ptr(lens), ptr(poff), ptr(lens), ptr(self.targets),
                                ptr(self.weights), sentinel, ptr(tgt), ptr(wts), st), "gee_span_copy")
        ns = (T + 1) * H
        check(lib.gee_span_copy(ns, ptr(src_first), ptr(src_len), ptr(t_first), ptr(dst_len), ptr(self.targets), None,
                                sentinel, ptr(tgt), None, st), "gee_span_copy")
        if wts is not None:
            check(lib.gee_span_copy(ns, ptr(src_first), ptr(src_len), ptr(r_first_o), ptr(dst_len), None,
                                    ptr(self.weights), sentinel, None, ptr(wts), st), "gee_span_copy")
        # 16-arc groups: tile-major position -> row-major position
        ng = dst_len // 16
        gstart = torch.cumsum(ng, 0) - ng
        gdst = torch.arange(int(ng.sum().item()), dtype=torch.int64, device=dev)
        gdst -= torch.repeat_interleave(gstart, ng)
        gdst += torch.repeat_interleave(r_first_o // 16, ng)
        self.group_dst = gdst.to(torch.int32)
        del gdst, ng, gstart
        seg_tot = dst_len.view(T + 1, H).sum(1)
        starts = torch.cumsum(seg_tot, 0) - seg_tot + light16  # tail, tile 0, ..., tile T-1
        self.tile_start = torch.cat([starts[1:], torch.tensor([total], dtype=torch.int64, device=dev)]).contiguous()
        self.light_arcs = light16
        self.l2_arcs = int(starts[1].item())  # light rows + the heavy tail
        self.n_tiles, self.tile_slots = T, ts
        row_len = rp.sum(1).cpu()
        row_first = r_first[:, 0].cpu()
        torch.cuda.current_stream(dev).synchronize()
        self.offsets, self.targets, self.weights = poff, tgt, wts
        self._owns_targets = self._owns_weights = True
        self._make_items(self.heavy_rows, row_first, row_len)
        ends = self.offsets[torch.arange(0, n + 32, 32, device=dev).clamp_(max=n)]
        self.max_block_arcs = int((ends[1:] - ends[:-1]).max().item()) if n else 0
        self.heavy_layout = "tiles"
        return True

    def _own_pull_arrays(self):
        """Private copies of the pull targets / weights before they are
        rewritten in place (hot encoding, row sort): never the caller's
        tensors, never the push layout's."""
        shared = lambda a, b: a is not None and b is not None and a.data_ptr() == b.data_ptr()  # noqa: E731
        if not self._owns_targets or shared(self.targets, self.dst):
            self.targets = self.targets.clone()
            self._owns_targets = True
        if self.weights is not None and (not self._owns_weights or shared(self.weights, self.w)):
            self.weights = self.weights.clone()
            self._owns_weights = True

    def _sort_rows(self):
        """Sort each row's arcs by label-table slot (graph preparation; the
        pull's integer sums do not depend on arc order)."""
        if self.arcs == 0:
            return
        self._own_pull_arrays()
        check(lib.gee_sort_rows(ptr(self.offsets), self.n, ptr(self.targets), ptr(self.weights), _stream()),
              "gee_sort_rows")

    @property
    def arcs(self):
        return 0 if self.targets is None else int(self.targets.numel())

    @property
    def has_pull(self):
        return self.offsets is not None

    @property
    def has_push(self):
        return self.src is not None

    @property
    def weighted(self):
        return (self.weights is not None) if self.has_pull else (self.w is not None)

    def csr_bytes(self):
        b = 0
        for t in (self.offsets, self.targets, self.weights):
            if t is not None:
                b += t.numel() * t.element_size()
        return b


# Fixed-point pull is accepted when its worst per-term relative rounding is
# 10x inside the 1e-4 parity bound.
PULL_REL_ERR_MAX = 1e-5


class Embedder:
    """Reusable device state for one (n, k): projection buffers, the label
    table and the pull slot buffer.  `project` + `pull`/`push` is one edge
    pass; nothing is allocated on those calls once warm."""

    def __init__(self, n, k, device=None):
        self.device = require_cuda(device)
        self.n, self.k = int(n), int(k)
        if self.k < 1:
            raise ValidationError("class count k must be positive")
        dev = self.device
        self.counts = torch.zeros(self.k + 1, dtype=torch.int64, device=dev)
        self.inv32 = torch.zeros(self.k + 1, dtype=torch.float32, device=dev)
        self.inv64 = torch.zeros(self.k + 1, dtype=torch.float64, device=dev)
        self.bad = torch.zeros(1, dtype=torch.int64, device=dev)
        self.table = None
        self.table_n_hot = None  # n_hot the current table was built with
        self.cls = None  # class stream of the split pull
        self.mega_acc = None  # mega-row partial sums (heavy items)
        self.counter = torch.zeros(1, dtype=torch.int64, device=dev)  # heavy-item work counter
        self.phase_events = None  # list -> (phase, cuda event) after each phase (bench)
        self.launches = 0  # our kernels launched so far (bench accounting)

    def _ensure_table(self, n_hot):
        need = int(lib.gee_label_table_bytes(self.n, n_hot, self.k))
        if self.table is None or self.table.numel() < need:
            self.table = torch.empty(need, dtype=torch.uint8, device=self.device)

    # ------------------------------------------------------------------ K1
    def project(self, labels_d, validate=True, g=None, inv=None):
        """Histogram + inv + label table (build_projection).  With a graph
        whose pull layout has a hot tier, the table carries its hot prefix.
        ``inv`` (float64[k+1], device or host) replaces the per-class values
        1/count: a caller-supplied ProjectionMatrix (encoder.py:116,155)."""
        if labels_d.numel() != self.n:
            raise ValidationError(f"graph has {self.n} nodes but labels have {labels_d.numel()}")
        hot_rank = g.hot_rank if (g is not None and g.hot_rank is not None) else None
        compact = g is not None and getattr(g, "hot_bits", None) is not None and g.n_hot > 0
        n_hot = g.n_hot if (hot_rank is not None or compact) else 0
        self._ensure_table(n_hot)
        if compact:
            check(lib.gee_build_projection_hotc(ptr(labels_d), self.n, self.k, ptr(self.counts), ptr(self.inv32),
                                                ptr(self.inv64), ptr(self.table), ptr(g.hot_bits), ptr(g.hot_pref),
                                                ptr(g.hot_list), n_hot, ptr(self.bad), _stream()),
                  "gee_build_projection_hotc")
        else:
            check(lib.gee_build_projection(ptr(labels_d), self.n, self.k, ptr(self.counts), ptr(self.inv32),
                                           ptr(self.inv64), ptr(self.table), ptr(hot_rank), n_hot, ptr(self.bad),
                                           _stream()), "gee_build_projection")
        self._mark("project", 2)
        self.table_n_hot = n_hot
        if inv is not None:
            self.inv64.copy_(torch.as_tensor(inv, dtype=torch.float64))
            self.inv32.copy_(self.inv64)
        if validate and int(self.bad.item()):
            raise ValidationError(f"{int(self.bad.item())} labels outside [0, {self.k}]")
        return self.counts

    def project_sharded(self, labels_d, g, count_lo, count_hi, reduce_counts):
        """The histogram sharded over row-range ranks: the
        label table still receives every label, but this rank counts only
        nodes [count_lo, count_hi); ``reduce_counts(counts)`` sums the k+1
        int64 counts over the ranks in place (one all-reduce), then inv."""
        if labels_d.numel() != self.n:
            raise ValidationError(f"graph has {self.n} nodes but labels have {labels_d.numel()}")
        if g is not None and g.hot_rank is not None and getattr(g, "hot_bits", None) is None:
            g.compact_hot()
        compact = g is not None and getattr(g, "hot_bits", None) is not None and g.n_hot > 0
        n_hot = g.n_hot if compact else 0
        self._ensure_table(n_hot)
        check(lib.gee_build_projection_sharded(
            ptr(labels_d), self.n, self.k, ptr(self.counts), ptr(self.table), ptr(g.hot_bits) if compact else None,
            ptr(g.hot_pref) if compact else None, ptr(g.hot_list) if compact else None, n_hot, int(count_lo),
            int(count_hi), ptr(self.bad), _stream()), "gee_build_projection_sharded")
        reduce_counts(self.counts)
        check(lib.gee_projection_inv(ptr(self.counts), self.k, ptr(self.inv32), ptr(self.inv64), _stream()),
              "gee_projection_inv")
        self._mark("project", 2)
        self.table_n_hot = n_hot
        return self.counts

    # ------------------------------------------------------------------ K4
    def new_z(self):
        return torch.empty((self.n, self.k), dtype=torch.float32, device=self.device)

    def reducer_for(self, g, z=None):
        """Which pull kernels run: "blocks" (class stream + 32-row block
        reducer + heavy items, k <= 255) or "wide" (label gather fused with a
        per-row window, any k).  Both are exact and give the same bits."""
        if self.k > 255 or not g.padded or g.max_block_arcs >= 2**31:
            return "wide"
        if z is not None and z.data_ptr() % 16:
            return "wide"
        return "blocks"

    def pull(self, g: DeviceGraph, z=None):
        if not g.has_pull:
            raise ValidationError("graph has no pull (symmetric CSR) layout")
        if g.n_nodes != self.n:
            raise ValidationError(f"graph has {g.n_nodes} nodes but labels have {self.n}")
        if g.weighted and g.rel_err > PULL_REL_ERR_MAX:
            raise ValidationError(
                f"weights span too wide a range for the exact fixed-point pull "
                f"(rounding bound {g.rel_err:.2e}); use variant='push'")
        if g.hot_k != self.k:
            raise ValidationError("call graph.prepare_hot(k) before the pull (Embedder.embed does)")
        if self.table_n_hot != g.n_hot:
            raise ValidationError("label table does not match the graph's hot tier: call project(labels, g=graph)")
        if z is None:
            z = torch.empty((g.n, self.k), dtype=torch.float32, device=self.device)
        if self.reducer_for(g, z) == "wide":
            check(lib.gee_reduce_wide(ptr(g.offsets), g.n, ptr(g.targets), ptr(g.weights), ptr(self.table), self.k,
                                      g.scale_exp, ptr(self.inv64), ptr(g.heavy_rows), g.n_heavy, ptr(z), _stream()),
                  "gee_reduce_wide")
            self._mark("wide", 1 + (1 if g.n_heavy else 0))
            return z
        # split pass: class stream (random gathers, full occupancy), then the
        # gather-free segmented reduction (light rows by 32-row blocks, heavy
        # rows as work items)
        if self.cls is None or self.cls.numel() < g.arcs + 64:
            self.cls = torch.empty(g.arcs + 64, dtype=torch.uint8, device=self.device)
        tiles = g.heavy_layout == "tiles"
        # light rows alone take a 128 KB head (no hub rows' lines to merge in L1):
        # C4 0 / 64 / 96 / 112 / 128 / 144 / 160 KB: 5.10 / 4.89 / 4.89 / 4.77 / 4.73 / 5.14 / 5.04 ms
        check(lib.gee_gather_labels_head(ptr(g.targets), g.light_arcs if tiles else g.arcs, ptr(self.table), g.n_hot,
                                         self.k, 131072 if tiles else -1, ptr(self.cls), _stream()),
              "gee_gather_labels")
        self._mark("gather", 1)
        if tiles:
            check(lib.gee_gather_scatter(ptr(g.targets), g.light_arcs, g.l2_arcs, g.light_arcs, ptr(g.group_dst),
                                         ptr(self.table), self.k, ptr(self.cls), _stream()), "gee_gather_scatter")
            check(lib.gee_gather_tiles(ptr(g.targets), ptr(g.tile_start), g.n_tiles, g.light_arcs, ptr(g.group_dst),
                                       ptr(self.table), g.n_hot + self.n + 1, g.tile_slots, self.k, ptr(self.cls),
                                       _stream()), "gee_gather_tiles")
            self._mark("tiles", 2 if g.l2_arcs > g.light_arcs else 1)
        if tiles:  # no heavy row left in the CSR: the skipping logic is compiled out
            check(lib.gee_reduce_blocks_short(ptr(g.offsets), g.n, ptr(self.cls), ptr(g.weights), g.scale_exp,
                                              ptr(self.inv64), self.k, ptr(g.short_rows) if g.short_arcs else None,
                                              g.short_arcs, ptr(z), _stream()), "gee_reduce_blocks_short")
        else:
            check(lib.gee_reduce_blocks_pad8(ptr(g.offsets), g.n, ptr(self.cls), ptr(g.weights), g.scale_exp,
                                             ptr(self.inv64), self.k, g.HEAVY_ARCS, ptr(z), _stream()),
                  "gee_reduce_blocks_pad8")
        self._mark("blocks", 1)
        if g.n_mega and (self.mega_acc is None or self.mega_acc.numel() < g.n_mega * self.k):
            self.mega_acc = torch.zeros(g.n_mega * self.k, dtype=torch.int64, device=self.device)
        check(lib.gee_reduce_heavy(ptr(self.cls), ptr(g.weights), g.arcs, g.scale_exp, ptr(self.inv64), self.k,
                                   ptr(g.item_first), ptr(g.item_end), ptr(g.item_row), ptr(g.item_slot), g.n_items,
                                   ptr(g.mega_rows), g.n_mega, ptr(self.mega_acc) if g.n_mega else None,
                                   ptr(self.counter), ptr(z), _stream()), "gee_reduce_heavy")
        self._mark("heavy", (1 if g.n_items else 0) + (1 if g.n_mega else 0))
        return z

    def _mark(self, phase, launches):
        """Phase bookkeeping for measurement: kernels launched, and a CUDA
        event on the current stream when `phase_events` is a list."""
        self.launches += launches
        if self.phase_events is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(torch.cuda.current_stream(self.device))
            self.phase_events.append((phase, ev))

    # ------------------------------------------------------------------ K3
    def push(self, g: DeviceGraph, z=None, precombine=False, zero=True):
        if not g.has_push:
            raise ValidationError("graph has no push (COO) layout")
        if g.n_nodes != self.n:
            raise ValidationError(f"graph has {g.n_nodes} nodes but labels have {self.n}")
        if self.table_n_hot is None:
            raise ValidationError("call project(labels) before the push")
        z = self.new_z() if z is None else z
        flags = (_lib.GEE_ZERO_Z if zero else 0) | (_lib.GEE_SOURCE_ONLY if g.coo_source_only else 0)
        if precombine:
            flags |= _lib.GEE_PRECOMBINE
        check(lib.gee_embed_coo(ptr(g.src), ptr(g.dst), ptr(g.w), int(g.src.numel()), ptr(self.table),
                                self.table_n_hot, ptr(self.inv32), g.n, self.k, ptr(z), flags, _stream()),
              "gee_embed_coo")
        self._mark("push", 2 if zero else 1)
        return z

    def embed(self, g: DeviceGraph, labels_d, variant="auto", z=None, validate=True, inv=None):
        """One edge pass: projection then the chosen edge map."""
        v = choose_variant(g, variant)
        if v == "pull":
            g.prepare_hot(self.k)
        self.project(labels_d, validate=validate, g=g if v == "pull" else None, inv=inv)
        return self.pull(g, z) if v == "pull" else self.push(g, z)


    def capture(self, g: DeviceGraph, labels_d, z, variant="pull"):
        """Record one edge pass (histogram + the edge map into z) as a CUDA
        graph; ``graph.replay()`` then re-runs it on the current contents of
        ``labels_d`` with one launch from the host.  Worth it where launches
        dominate (C1: 140K edges, six kernels); the buffers stay bound to the
        graph.  The pass runs once eagerly first (kernel attributes, scratch
        sizing, label validation)."""
        v = choose_variant(g, variant)
        if v == "pull":
            g.prepare_hot(self.k)
        self.project(labels_d, validate=True, g=g if v == "pull" else None)
        (self.pull if v == "pull" else self.push)(g, z)
        if g.n_mega and self.mega_acc is None:
            self.mega_acc = torch.zeros(g.n_mega * self.k, dtype=torch.int64, device=self.device)
        torch.cuda.synchronize(self.device)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            self.project(labels_d, validate=False, g=g if v == "pull" else None)
            (self.pull if v == "pull" else self.push)(g, z)
        return graph


def choose_variant(g: DeviceGraph, variant="auto"):
    """Pull wherever its layout exists and its fixed point is exact enough.

    Measured on B200 (profiles/): pull writes each Z row once and reads
    labels through L1/L2 with no Z read-modify-write; push pays a 32 B
    sector RMW per red.global once Z outgrows L2 (~20 G red/s).
    """
    if variant not in ("auto", "pull", "push"):
        raise ValidationError(f"unknown variant {variant!r}")
    if variant != "auto":
        return variant
    if g.has_pull and (not g.weighted or g.rel_err <= PULL_REL_ERR_MAX):
        return "pull"
    if g.has_push:
        return "push"
    return "pull"


def build_csr(el, stable=True):
    """graph.build_csr on the GPU (mirror arcs for undirected lists)."""
    from .graph import CsrGraph, _is_torch

    dev = require_cuda(el.src.device if _is_torch(el.src) and el.src.is_cuda else None)
    on_host = not (_is_torch(el.src) and el.src.is_cuda)
    src_d = to_device(el.src, torch.int32, dev)
    dst_d = to_device(el.dst, torch.int32, dev)
    w_d = to_device(el.w, torch.float32, dev)
    s, n = el.s, el.n
    sym = 0 if el.directed else 1
    arcs = s * (2 if sym else 1)
    offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
    targets = torch.empty(arcs, dtype=torch.int32, device=dev)
    weights = torch.empty(arcs, dtype=torch.float32, device=dev) if w_d is not None else None
    check(lib.gee_build_csr(ptr(src_d), ptr(dst_d), ptr(w_d), s, n, sym, 1 if stable else 0, ptr(offsets),
                            ptr(targets), ptr(weights), _stream()), "gee_build_csr")
    if on_host:
        offsets, targets = offsets.cpu().numpy(), targets.cpu().numpy()
        weights = weights.cpu().numpy() if weights is not None else None
    return CsrGraph(n=n, offsets=offsets, targets=targets, weights=weights, directed=el.directed)
