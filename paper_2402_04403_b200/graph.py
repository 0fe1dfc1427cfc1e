"""Graph containers and CSR construction (mirror of the reference graph.py).

Same names, fields and validation rules as the reference
(/root/reference/pkg/src/gee/graph.py), with the edge pass's device dtypes:
int32 endpoints (the reference's CSR limit is already int32,
graph.py:14-15,166-167), float32 weights, and ``w=None`` for unit weights.
Arrays may be numpy (host) or torch tensors (host or CUDA); validation runs
where the data lives.
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import ValidationError

# CSR targets are int32 (graph.py:14-15).
MAX_NODES = np.iinfo(np.int32).max


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _as_index(a, name):
    if _is_torch(a):
        import torch

        if a.dtype != torch.int32:
            if a.numel() and (int(a.min()) < np.iinfo(np.int32).min or int(a.max()) > MAX_NODES):
                raise ValidationError(f"{name} values do not fit int32")
            a = a.to(torch.int32)
        return a.contiguous().reshape(-1)
    a = np.asarray(a)
    if a.size == 0:
        return np.zeros(0, dtype=np.int32)
    if not np.issubdtype(a.dtype, np.integer):
        if not np.all(np.isfinite(a)) or not np.all(a == np.floor(a)):
            raise ValidationError(f"{name} must hold integers")
    if a.dtype != np.int32:
        if a.min() < np.iinfo(np.int32).min or a.max() > MAX_NODES:
            raise ValidationError(f"{name} values do not fit int32")
    return np.ascontiguousarray(a, dtype=np.int32).reshape(-1)


_F32_MAX = float(np.finfo(np.float32).max)
_F32_TINY = float(np.finfo(np.float32).tiny)  # smallest normal float32


def _check_f32_range(finite, absmax, absmin_nz, name, what):
    """Checks on the caller's dtype BEFORE narrowing to float32: a finite
    f64 weight above FLT_MAX would become inf, and one below the normal
    range would lose its precision (or vanish) -- both would break parity
    with the reference's f64 pass without a diagnostic."""
    if not finite:
        raise ValidationError(f"{what} weights must be finite")
    if absmax > _F32_MAX:
        raise ValidationError(f"{name}: |weight| {absmax:.6g} exceeds the float32 range of the edge pass")
    if 0.0 < absmin_nz < _F32_TINY:
        raise ValidationError(f"{name}: nonzero |weight| {absmin_nz:.6g} is below the normal float32 range "
                              f"({_F32_TINY:.6g}) of the edge pass")


def _as_weights(w, name, what="edge"):
    if w is None:
        return None
    if _is_torch(w):
        import torch

        w = w.contiguous().reshape(-1)
        if w.dtype != torch.float32 and w.numel():
            a = w.to(torch.float64).abs()
            nz = a[a > 0]
            _check_f32_range(bool(torch.isfinite(a).all()), float(a.max()),
                             float(nz.min()) if nz.numel() else 0.0, name, what)
        return w.to(torch.float32)
    w = np.asarray(w).reshape(-1)
    if w.dtype != np.float32 and w.size:
        a = np.abs(w.astype(np.float64))
        nz = a[a > 0]
        _check_f32_range(bool(np.isfinite(a).all()), float(a.max()), float(nz.min()) if nz.size else 0.0, name, what)
    return np.ascontiguousarray(w, dtype=np.float32)


def _minmax(a):
    if _is_torch(a):
        return int(a.min()), int(a.max())
    return int(a.min()), int(a.max())


def _all_finite(w):
    if _is_torch(w):
        import torch

        return bool(torch.isfinite(w).all())
    return bool(np.isfinite(w).all())


def _all_ones(w):
    if _is_torch(w):
        return bool((w == 1.0).all())
    return bool(np.all(w == 1.0))


def _length(a):
    return int(a.shape[0])


@dataclass(eq=False)
class EdgeList:
    """Flat edge list: s triples (src, dst, weight) over nodes 0..n-1.

    Mirrors graph.py:18-51.  ``w=None`` means unit weights (the reference
    stores explicit ones).  ``directed=False`` means each listed edge stands
    for both directions; the list itself stores each edge once.  The edge
    pass applies both updates per listed edge either way
    (encoder.py:106-120); ``directed`` only selects CSR storage.
    """

    n: int
    src: object
    dst: object
    w: object = None
    directed: bool = True

    def __post_init__(self):
        self.n = int(self.n)
        if self.n < 0:
            raise ValidationError("node count must be nonnegative")
        if self.n > MAX_NODES:
            raise ValidationError(f"node count {self.n} exceeds int32 limit {MAX_NODES}")
        self.src = _as_index(self.src, "src")
        self.dst = _as_index(self.dst, "dst")
        self.w = _as_weights(self.w, "w")
        if _length(self.src) != _length(self.dst) or (self.w is not None and _length(self.w) != _length(self.src)):
            raise ValidationError("src, dst and w must have equal length")
        if self.s:
            lo_s, hi_s = _minmax(self.src)
            lo_d, hi_d = _minmax(self.dst)
            if min(lo_s, lo_d) < 0 or max(hi_s, hi_d) >= self.n:
                raise ValidationError(f"edge endpoint out of range [0, {self.n})")
            if self.w is not None and not _all_finite(self.w):
                raise ValidationError("edge weights must be finite")
        if self.w is not None and (self.s == 0 or _all_ones(self.w)):
            self.w = None  # unit weights: the kernels skip the weight stream

    @property
    def s(self) -> int:
        return _length(self.src)

    @property
    def unit_weights(self) -> bool:
        return self.w is None

    def weights(self):
        """Per-edge weights as an array (ones when unit)."""
        if self.w is not None:
            return self.w
        if _is_torch(self.src):
            import torch

            return torch.ones(self.s, dtype=torch.float32, device=self.src.device)
        return np.ones(self.s, dtype=np.float32)


@dataclass(eq=False)
class CsrGraph:
    """Compressed sparse row adjacency with per-arc weights (graph.py:54-91).

    An undirected edge list is stored symmetrically: both (u, v) and (v, u)
    appear as arcs with equal weight.  ``weights=None`` means unit weights.
    """

    n: int
    offsets: object
    targets: object
    weights: object = None
    directed: bool = True
    unit_weights: bool = field(init=False)

    def __post_init__(self):
        self.n = int(self.n)
        if _is_torch(self.offsets):
            import torch

            self.offsets = self.offsets.to(torch.int64).contiguous().reshape(-1)
        else:
            self.offsets = np.ascontiguousarray(self.offsets, dtype=np.int64).reshape(-1)
        self.targets = _as_index(self.targets, "targets")
        self.weights = _as_weights(self.weights, "weights", "arc")
        if self.n > MAX_NODES:
            raise ValidationError(f"node count {self.n} exceeds CSR limit {MAX_NODES}")
        if _length(self.offsets) != self.n + 1:
            raise ValidationError("offsets must have length n + 1")
        if int(self.offsets[0]) != 0 or int(self.offsets[-1]) != self.s:
            raise ValidationError("offsets must start at 0 and end at the arc count")
        if self.n and _is_torch(self.offsets):
            if bool((self.offsets[1:] < self.offsets[:-1]).any()):
                raise ValidationError("offsets must be nondecreasing")
        elif self.n and np.any(np.diff(self.offsets) < 0):
            raise ValidationError("offsets must be nondecreasing")
        if self.weights is not None and _length(self.weights) != self.s:
            raise ValidationError("targets and weights must have equal length")
        if self.s:
            lo, hi = _minmax(self.targets)
            if lo < 0 or hi >= self.n:
                raise ValidationError(f"arc target out of range [0, {self.n})")
            if self.weights is not None and not _all_finite(self.weights):
                raise ValidationError("arc weights must be finite")
        if self.weights is not None and (self.s == 0 or _all_ones(self.weights)):
            self.weights = None
        self.unit_weights = self.weights is None

    @property
    def s(self) -> int:
        """Number of stored arcs (2x the edge count for undirected input)."""
        return _length(self.targets)


def build_csr(el: EdgeList, stable=True) -> CsrGraph:
    """Counting-sort an edge list into CSR form on the GPU (graph.py:159-184).

    Directed input maps each edge to one arc; undirected input inserts the
    mirror arc immediately after the original.  With ``stable=True`` (the
    reference's order) a node's arc range keeps the input edge order; with
    ``stable=False`` arc order within a row is unspecified (cheaper; the
    pull edge pass is order-independent).  Returns a CsrGraph whose arrays
    live where the edge list lives (host arrays in -> host arrays out).
    """
    from . import device

    return device.build_csr(el, stable=stable)


def generate_erdos_renyi(n, s, seed, device=None) -> EdgeList:
    """G(n, s): exactly s directed unit-weight edges with uniform endpoints.

    Same contract as graph.py:187-201 (self-loops and duplicates kept,
    deterministic in (n, s, seed)).  With ``device=None`` the endpoints are
    the reference's own numpy stream (default_rng(seed).integers twice), so
    a seed gives the reference's edge sequence; with a CUDA ``device`` they
    come from the counter-based generator in gee_synth.cu (a different
    stream, generated in HBM at memory speed).
    """
    if n < 1:
        raise ValidationError("n must be at least 1")
    if s < 0:
        raise ValidationError("s must be nonnegative")
    if device is None:
        if n - 1 > MAX_NODES:
            raise ValidationError(f"node count {n} exceeds int32 limit {MAX_NODES}")
        rng = np.random.default_rng(seed)
        src = rng.integers(0, n, size=s, dtype=np.int64)
        dst = rng.integers(0, n, size=s, dtype=np.int64)
        return EdgeList(n=n, src=src, dst=dst, w=None, directed=True)
    from . import synth

    src, dst, _ = synth.er_edges(n, s, seed, weighted=False, device=device)
    return EdgeList(n=n, src=src, dst=dst, w=None, directed=True)
