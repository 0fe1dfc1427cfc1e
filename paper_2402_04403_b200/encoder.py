"""One-hot graph encoder embedding on B200 (mirror of the reference encoder.py).

Entry points keep the reference's names, arguments and error behaviour
(/root/reference/pkg/src/gee/encoder.py); the arithmetic runs in
libgee_b200.so:

  build_projection  encoder.py:80-103   K1 histogram kernel (bit-exact counts)
  embed_serial      encoder.py:106-120  one pass over the listed edges
  embed_parallel    encoder.py:123-194  one pass over a stored CsrGraph
  embed             north-star entry: arrays in, n x K Z out

Z is float32 (the reference's is float64).  Parity
with the f64 oracle: max relative error <= 1e-4 per entry, zeros exact.
The pull variant (default) accumulates exactly in integers, so it is
bitwise reproducible like embed_serial; the push variant uses fp32
red.global atomics (order-dependent rounding).
"""

import enum
import logging
import threading

import numpy as np

from .errors import ValidationError
from .graph import CsrGraph, EdgeList, _is_torch
from .labeling import LabelVector

logger = logging.getLogger(__name__)


class EdgeAccounting(enum.Enum):
    """Per-arc update rule that makes the arc pass match the edge-list pass
    (encoder.py:37-48): directed storage applies both updates per arc,
    symmetric storage only the source-side one."""

    BOTH_ENDPOINTS = "both"
    SOURCE_ONLY = "source"


def edge_accounting(g: CsrGraph, directed=None) -> EdgeAccounting:
    """Pick the update rule for a stored graph (encoder.py:51-55)."""
    if directed is None:
        directed = g.directed
    return EdgeAccounting.BOTH_ENDPOINTS if directed else EdgeAccounting.SOURCE_ONLY


class ProjectionMatrix:
    """The n x K projection W stored as one scalar per node (encoder.py:58-77).

    ``counts`` (int64[k+1], bin 0 = unlabeled) comes from the GPU histogram.
    """

    def __init__(self, n, k, row_value, label, counts=None):
        self.n = n
        self.k = k
        self.row_value = row_value  # float64[n]
        self.label = label  # int32[n], 0 = unknown
        self.counts = counts

    def to_dense(self) -> np.ndarray:
        """Materialize W as a dense n x K array (small graphs / tests)."""
        w = np.zeros((self.n, self.k))
        idx = np.nonzero(self.label)[0]
        w[idx, self.label[idx] - 1] = self.row_value[idx]
        return w


def _device_for(*arrays):
    for a in arrays:
        if _is_torch(a) and a.is_cuda:
            return a.device
    return None


def _projection_tables(y: LabelVector):
    """Run K1 on the labels; return (counts int64[k+1], inv f64[k+1]) on host."""
    import torch

    from .device import Embedder, to_device, require_cuda

    dev = require_cuda(_device_for(y.labels))
    lab = to_device(y.labels, torch.int32, dev)
    emb = Embedder(y.n, y.k, dev)
    emb.project(lab)
    return emb.counts.cpu().numpy(), emb.inv64.cpu().numpy()


def _counts_on_device(y: LabelVector) -> np.ndarray:
    return _projection_tables(y)[0]


def build_projection(y: LabelVector) -> ProjectionMatrix:
    """Construct W from the labels: W[i, Y[i]-1] = 1 / count(Y == Y[i]).

    Counts come from the GPU histogram (bit-exact with np.bincount); empty
    classes and all-unlabeled inputs are logged as in encoder.py:88-94.
    """
    counts, inv = _projection_tables(y)
    labeled = int(y.n - counts[0])
    if labeled == 0:
        logger.warning("no labeled nodes: the embedding will be identically zero")
    else:
        empty = np.nonzero(counts[1:] == 0)[0] + 1
        if empty.size:
            logger.warning("%d of %d classes have no members", empty.size, y.k)
    lab = y.labels.cpu().numpy() if _is_torch(y.labels) else y.labels
    return ProjectionMatrix(n=y.n, k=y.k, row_value=inv[lab], label=lab.astype(np.int32), counts=counts)


def _check_out(out, n, k):
    """Validate a caller-owned output buffer (encoder.py:156-163)."""
    if out is None:
        return None
    if _is_torch(out):
        import torch

        if tuple(out.shape) != (n, k) or out.dtype != torch.float32 or not out.is_contiguous() or not out.is_cuda:
            raise ValidationError(f"out must be a contiguous float32 CUDA tensor of shape ({n}, {k})")
        return out
    if (
        not isinstance(out, np.ndarray)
        or out.shape != (n, k)
        or out.dtype not in (np.float32, np.float64)
        or not out.flags.c_contiguous
    ):
        raise ValidationError(f"out must be a C-contiguous float32/float64 array of shape ({n}, {k})")
    return out


def _finish(z_d, out, host):
    """Deliver the device result into `out` or a fresh host/device array."""
    if out is not None:
        if _is_torch(out):
            if out.data_ptr() != z_d.data_ptr():
                out.copy_(z_d)
            return out
        out[...] = z_d.cpu().numpy()
        return out
    return z_d.cpu().numpy() if host else z_d


def _validate_projection(projection, n, k):
    if projection is not None and (projection.n != n or projection.k != k):
        raise ValidationError(f"projection is ({projection.n}, {projection.k}) but the pass is ({n}, {k})")


def _projection_inv(projection, labels, k):
    """Per-class values of a caller-supplied ProjectionMatrix.

    The reference reads W as (labels, row_value) per node: embed_serial pairs
    y.labels with projection.row_value (encoder.py:116-119), embed_parallel
    reads projection.label and projection.row_value (encoder.py:155,
    :180-181).  The edge pass here sums weights per (row, class) and scales
    each class once, so row_value must be one value per class among the
    labeled nodes (true of every build_projection output, whatever the
    counts); that value replaces 1/count.  Per-node values that differ
    within a class raise ValidationError instead of being ignored."""
    import torch

    lab = torch.as_tensor(labels).to(torch.int64).reshape(-1)
    rv = torch.as_tensor(projection.row_value, dtype=torch.float64, device=lab.device).reshape(-1)
    if rv.numel() != lab.numel():
        raise ValidationError(f"projection.row_value has {rv.numel()} entries for {lab.numel()} nodes")
    keep = (lab > 0) & (lab <= k)
    lab, rv = lab[keep], rv[keep]
    if not bool(torch.isfinite(rv).all()):
        raise ValidationError("projection.row_value must be finite")
    hi = torch.zeros(k + 1, dtype=torch.float64, device=lab.device).scatter_reduce_(0, lab, rv, "amax",
                                                                                     include_self=False)
    lo = torch.zeros(k + 1, dtype=torch.float64, device=lab.device).scatter_reduce_(0, lab, rv, "amin",
                                                                                     include_self=False)
    if not bool(torch.equal(hi, lo)):
        raise ValidationError("projection.row_value must be constant within each class: the GPU edge pass "
                              "scales per (row, class) sum, not per node")
    hi[0] = 0.0
    return hi


# ---------------------------------------------------------------- variants
# Which edge map a call runs ("auto").  embed_serial is the reference's
# bit-reproducible oracle (encoder.py:106-113), so it always takes the exact
# integer pull.  embed_parallel's reference pass is itself order-dependent
# (CAS f64 atomics, encoder.py:139-142), so it takes whichever variant the
# measured table says is faster for a whole call of that size: the push
# needs no graph preparation (CSR mirror, hot tier, row sort, padding) and
# wins on small graphs (profiles/r02_variant_table.json, one B200, host
# arrays in and out: push 2.9 vs pull 5.0 ms at 2M arcs, 23.6 vs 26.4 ms at
# 6M, even at 20M-60M arcs, where the resident pass then favours the pull).
PUSH_MAX_ARCS = 1 << 23

_last = threading.local()


def last_pass():
    """Variant and kernels of the most recent embed_* call on this thread:
    {"variant": "pull"|"push", "reducer": "blocks"|"wide"|"prepared"|None,
    "reason": why}."""
    return dict(getattr(_last, "info", {}))


def _record(variant, reducer, reason):
    _last.info = dict(variant=variant, reducer=reducer, reason=reason)
    logger.debug("edge pass: variant=%s reducer=%s (%s)", variant, reducer, reason)


def _gate_push_warning(rel_err):
    logger.warning(
        "weights span too wide a range for the exact fixed-point pull (worst per-term rounding %.2e > %.0e): "
        "running the push variant (fp32 atomics; Z is not bit-stable run to run)", rel_err, 1e-5)


def embed_serial(el: EdgeList, y: LabelVector, projection=None, *, variant="auto", out=None):
    """One pass over the listed edges (embed_serial, encoder.py:106-120).

    Every listed edge applies both updates, for directed and undirected
    lists alike.  The default pull variant is bitwise reproducible.
    """
    import torch

    from .device import PULL_REL_ERR_MAX, DeviceGraph, Embedder, require_cuda, to_device

    if el.n != y.n:
        raise ValidationError(f"graph has {el.n} nodes but labels have {y.n}")
    _validate_projection(projection, el.n, y.k)
    out = _check_out(out, el.n, y.k)
    dev = require_cuda(_device_for(el.src, y.labels, out))
    host = not (_is_torch(el.src) and el.src.is_cuda)
    if el.n == 0:
        return _finish(torch.zeros((0, y.k), dtype=torch.float32, device=dev), out, host)
    lab_d = to_device(y.labels, torch.int32, dev)
    inv = None if projection is None else _projection_inv(projection, lab_d, y.k)
    want = variant if variant != "auto" else "pull"
    reason = "requested" if variant != "auto" else "embed_serial is bit-reproducible: exact pull"
    g = DeviceGraph.from_edges(el.src, el.dst, el.w, el.n, device=dev, pull=(want == "pull"),
                               keep_coo=(want == "push"))
    if variant == "auto" and g.weighted and g.rel_err > PULL_REL_ERR_MAX:
        _gate_push_warning(g.rel_err)
        reason = f"fixed-point gate (rounding {g.rel_err:.2e})"
        g = DeviceGraph.from_edges(el.src, el.dst, el.w, el.n, device=dev, pull=False, keep_coo=True)
        want = "push"
    emb = Embedder(el.n, y.k, dev)
    z_d = out if (_is_torch(out)) else None
    z_d = emb.embed(g, lab_d, variant=want, z=z_d, inv=inv)
    _record(want, emb.reducer_for(g, z_d) if want == "pull" else None, reason)
    torch.cuda.current_stream().synchronize()
    return _finish(z_d, out, host)


def embed_parallel(
    g: CsrGraph,
    y: LabelVector,
    *,
    workers=None,
    atomics=True,
    accounting=None,
    projection=None,
    out=None,
    variant="auto",
):
    """Edge map over all arcs of a stored CsrGraph (encoder.py:123-194).

    ``g`` may also be a ``PreparedGraph`` (``prepare(g, k)``): graph
    preparation then happened once, outside the call, and the call streams
    the prepared layout from pinned host memory (or runs it from HBM) --
    the path for repeated passes over a large graph.

    ``workers`` is validated like the reference (>= 1) and otherwise
    ignored: the GPU kernels size their own grids.  ``atomics=False`` (the
    reference's unsafe mode for measuring atomic cost) selects the pull
    variant, which has no atomics on Z.  ``out`` may be a caller-owned
    (n, k) float32/float64 C-contiguous array (or float32 CUDA tensor) that
    is overwritten and returned.
    """
    import torch

    from .device import PULL_REL_ERR_MAX, DeviceGraph, Embedder, require_cuda, to_device
    from .prepared import PreparedGraph

    if g.n != y.n:
        raise ValidationError(f"graph has {g.n} nodes but labels have {y.n}")
    if workers is not None and workers < 1:
        raise ValidationError("workers must be at least 1")
    if isinstance(g, PreparedGraph):
        # graph preparation already done (prepare()): only the per-call pass
        if variant not in ("auto", "pull"):
            raise ValidationError("a prepared graph runs the pull variant")
        _validate_projection(projection, g.n, y.k)
        if projection is not None:
            y = LabelVector(labels=projection.label, k=y.k)
        out = _check_out(out, g.n, y.k)
        inv = None
        if projection is not None:
            inv = _projection_inv(projection, to_device(y.labels, torch.int32, g.device), y.k)
        res = g.run(y, out=out, inv=inv)
        _record("pull", "prepared", f"prepared graph ({g.residency} residency)")
        return res
    if accounting is None:
        accounting = edge_accounting(g)
    _validate_projection(projection, g.n, y.k)
    out = _check_out(out, g.n, y.k)
    if not atomics and variant == "auto":
        variant = "pull"
    dev = require_cuda(_device_for(g.targets, y.labels, out))
    host = not (_is_torch(g.targets) and g.targets.is_cuda)
    if g.n == 0 or y.k == 0:
        return _finish(torch.zeros((g.n, y.k), dtype=torch.float32, device=dev), out, host)
    symmetric = accounting is EdgeAccounting.SOURCE_ONLY
    labels = projection.label if projection is not None else y.labels
    lab_d = to_device(labels, torch.int32, dev)
    inv = None if projection is None else _projection_inv(projection, lab_d, y.k)
    arcs = int(g.targets.shape[0])
    if variant != "auto":
        want, reason = variant, "requested"
    elif not atomics:
        want, reason = "pull", "atomics=False: the atomic-free pull"
    elif arcs <= PUSH_MAX_ARCS:
        want, reason = "push", f"measured table: push for <= {PUSH_MAX_ARCS} arcs"
    else:
        want, reason = "pull", f"measured table: pull for > {PUSH_MAX_ARCS} arcs"
    dg = DeviceGraph.from_csr(g.offsets, g.targets, g.weights, g.n, symmetric, device=dev,
                              pull=want == "pull", keep_coo=want == "push")
    if variant == "auto" and want == "pull" and dg.weighted and dg.rel_err > PULL_REL_ERR_MAX:
        _gate_push_warning(dg.rel_err)
        reason = f"fixed-point gate (rounding {dg.rel_err:.2e})"
        dg = DeviceGraph.from_csr(g.offsets, g.targets, g.weights, g.n, symmetric, device=dev,
                                  pull=False, keep_coo=True)
        want = "push"
    emb = Embedder(g.n, y.k, dev)
    z_d = out if _is_torch(out) else None
    z_d = emb.embed(dg, lab_d, variant=want, z=z_d, inv=inv)
    _record(want, emb.reducer_for(dg, z_d) if want == "pull" else None, reason)
    torch.cuda.current_stream().synchronize()
    return _finish(z_d, out, host)


def embed(src, dst, labels, n, k, weights=None, directed=True, *, variant="auto", out=None):
    """North-star entry point: edge list + optional weights + labels in,
    n x K float32 Z out (host arrays in -> numpy out; CUDA tensors in ->
    CUDA tensor out)."""
    el = EdgeList(n=n, src=src, dst=dst, w=weights, directed=directed)
    y = LabelVector(labels=labels, k=k)
    return embed_serial(el, y, variant=variant, out=out)
