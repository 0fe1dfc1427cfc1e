"""Multi-GPU sharding of the edge pass (one process per GPU).

row-range ownership (default, no data-path collective)
    Node ranges [r_g, r_{g+1}) balanced by the estimated bytes each rank
    moves: its symmetric arcs (target + weight) plus its Z rows.  Every
    listed edge (u, v, w) becomes the half-edges u<-v (owner(u)) and v<-u
    (owner(v)) -- the symmetric CSR split by rows -- and each rank runs the
    pull kernel on its rows and writes its Z slice exactly once.  Labels
    (and so the histogram) are replicated: every rank reads all n labels.

edge-range (measured alternative)
    Contiguous slices of the listed edges; each rank pushes into a full
    fp32 Z partial and `reduce_scatter_tensor` (NCCL, sum) leaves each rank
    its row slice.  Moves (g-1)/g * n*K*4 bytes per rank over NVLink.

The planners are pure host functions (numpy) so they are tested on CPU
with gloo; the device parts go through libgee_b200.so.
"""

import numpy as np

from .errors import ValidationError


def plan_rows(offsets, world, k, weighted):
    """Row boundaries [b_0=0, ..., b_world=n] balancing arcs*(4+4w) + rows*4k.

    `offsets` is the full symmetric CSR offsets array (n+1, int64, host).
    Deterministic: every rank computes the same plan from the same offsets.
    """
    offsets = np.asarray(offsets, dtype=np.int64)
    n = offsets.size - 1
    if world < 1:
        raise ValidationError("world size must be >= 1")
    if n == 0:
        return np.zeros(world + 1, dtype=np.int64)
    arc_bytes = 4 + 4 * int(bool(weighted))
    # cumulative cost at row boundary r: arcs before r + rows before r
    cost = offsets * arc_bytes + np.arange(n + 1, dtype=np.int64) * (4 * k)
    total = cost[-1]
    targets = (np.arange(1, world, dtype=np.float64) * total / world)
    cuts = np.searchsorted(cost, targets, side="left").astype(np.int64)
    bounds = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    return np.maximum.accumulate(bounds)


def plan_edges(s, world):
    """Contiguous listed-edge slices [e_0=0, ..., e_world=s] for edge-range sharding."""
    return (np.arange(world + 1, dtype=np.int64) * s) // world


def build_row_shard(src, dst, w, n, world, rank, k=None):
    """This rank's pull layout from the full listed edge list on its GPU.

    Returns (DeviceGraph over local rows, row_lo, row_hi).  The graph's
    targets stay global node ids; rows are local (0 = row_lo).
    """
    import torch

    from . import _lib
    from ._lib import check, lib, ptr
    from .device import DeviceGraph

    dev = src.device
    s = int(src.numel())
    full = torch.empty(n + 1, dtype=torch.int64, device=dev)
    check(lib.gee_sym_offsets(ptr(src), ptr(dst), s, n, ptr(full), _lib.stream_handle()), "gee_sym_offsets")
    kk = k if k is not None else 1
    bounds = plan_rows(full.cpu().numpy(), world, kk, w is not None)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    arcs = int(full[hi].item() - full[lo].item())
    g = DeviceGraph(hi - lo, s, dev)
    g.offsets = torch.empty(hi - lo + 1, dtype=torch.int64, device=dev)
    g.targets = torch.empty(arcs, dtype=torch.int32, device=dev)
    g.weights = torch.empty(arcs, dtype=torch.float32, device=dev) if w is not None else None
    check(lib.gee_build_sym_csr_rows(ptr(src), ptr(dst), ptr(w), s, n, lo, hi, ptr(full), ptr(g.offsets),
                                     ptr(g.targets), ptr(g.weights), _lib.stream_handle()), "gee_build_sym_csr_rows")
    g._plan()
    g.n_nodes = n
    g.global_offsets = full  # global degrees for the hot-label plan (freed by prepare_hot)
    return g, lo, hi


def merge_weight_stats(stats):
    """Whole-graph weight statistics from per-shard (max_row_abs, max_abs,
    min_abs) triples: max, max, and min over the shards' nonzero minima."""
    stats = list(stats)
    mins = [s[2] for s in stats if s[2] > 0]
    return (max((s[0] for s in stats), default=0.0), max((s[1] for s in stats), default=0.0),
            min(mins) if mins else 0.0)


def unify_scale_distributed(g, group=None):
    """All ranks adopt the whole graph's fixed-point exponent (one 3-value
    all-reduce at graph preparation; nothing on the data path)."""
    import torch
    import torch.distributed as dist

    mx, mxa, mn = g.weight_stats()
    dev = g.device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    hi = torch.tensor([mx, mxa], dtype=torch.float64, device=dev)
    lo = torch.tensor([mn if mn > 0 else float("inf")], dtype=torch.float64, device=dev)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    mn_all = float(lo[0])
    g.adopt_scale((float(hi[0]), float(hi[1]), 0.0 if mn_all == float("inf") else mn_all))


def label_slice(n, world, rank):
    """[lo, hi): the nodes whose labels this rank counts in the sharded
    histogram (contiguous, n/world each)."""
    if world < 1 or not 0 <= rank < world:
        raise ValidationError("rank outside [0, world)")
    return (n * rank) // world, (n * (rank + 1)) // world


def allreduce_counts(counts, group=None):
    """Sum the per-rank class counts (k+1 int64) over the ranks, in place."""
    import torch.distributed as dist

    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def reduce_scatter_rows(z_partial, world, group=None):
    """Edge-range combine: sum the (n, k) partials across ranks and return
    this rank's contiguous row slice (rows padded to a multiple of world)."""
    import torch
    import torch.distributed as dist

    n, k = z_partial.shape
    per = -(-n // world)
    if per * world != n:
        pad = torch.zeros((per * world - n, k), dtype=z_partial.dtype, device=z_partial.device)
        z_partial = torch.cat([z_partial, pad])
    out = torch.empty((per, k), dtype=z_partial.dtype, device=z_partial.device)
    dist.reduce_scatter_tensor(out, z_partial.contiguous(), op=dist.ReduceOp.SUM, group=group)
    return out
