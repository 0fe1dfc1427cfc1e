"""Data formats of the reference, read and written by native code (libgee_io.so).

Mirrors the reference's IO functions with the same names, arguments, check
order and error text (files under /root/reference/pkg/src/gee):

  load_edge_list / write_edge_list          graph.py:94-156
  read_binary_cache / write_binary_cache    graph.py:204-235 (GEECSR1)
  load_labels / write_labels                labeling.py:33-84
  read_embedding / write_embedding          encoder.py:209-237 (GEEEMB1, csv)

The parsing and the byte work run in the multithreaded C++ library declared
in include/gee_io.h; this module allocates the arrays, calls it through
ctypes and applies the reference's value checks.  Arrays come back in the
edge pass's dtypes (int32 ids, float32 weights);
``device=`` stages a graph through pinned host memory onto a GPU.
"""

import ctypes
import os

import numpy as np

from .errors import FormatError, GeeError, ParseError, ValidationError
from .graph import MAX_NODES, CsrGraph, EdgeList, _is_torch
from .labeling import LabelVector

CACHE_MAGIC = b"GEECSR1\x00"  # graph.py:11
CACHE_VERSION = 1  # graph.py:12
EMB_MAGIC = b"GEEEMB1\x00"  # encoder.py:31

_PKG = os.path.dirname(os.path.abspath(__file__))
IO_LIB_PATH = os.path.join(_PKG, "libgee_io.so")

GEE_IO_OK, GEE_IO_ERR_OS, GEE_IO_ERR_PARSE, GEE_IO_ERR_FORMAT, GEE_IO_ERR_VALUE, GEE_IO_ERR_INVALID = range(6)

_vp, _i32, _i64, _int = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int
_cs = ctypes.c_char_p
_P_i64 = ctypes.POINTER(ctypes.c_int64)
_P_int = ctypes.POINTER(ctypes.c_int)

# every symbol include/gee_io.h declares
IO_SIGNATURES = {
    "gee_io_version": (_int, []),
    "gee_io_last_error": (_cs, []),
    "gee_io_last_errno": (_int, []),
    "gee_io_edges_parse": (_int, [_cs, _int, _int, ctypes.POINTER(_vp)]),
    "gee_io_edges_count": (_i64, [_vp]),
    "gee_io_edges_max_id": (_i64, [_vp]),
    "gee_io_edges_copy_i32": (_int, [_vp, _vp, _vp, _vp, _int]),
    "gee_io_edges_copy_i64": (_int, [_vp, _vp, _vp, _vp, _int]),
    "gee_io_edges_free": (None, [_vp]),
    "gee_io_edges_write": (_int, [_cs, _vp, _vp, _vp, _i64, _int]),
    "gee_io_labels_parse": (_int, [_cs, _int, ctypes.POINTER(_vp)]),
    "gee_io_labels_width": (_int, [_vp]),
    "gee_io_labels_rows": (_i64, [_vp]),
    "gee_io_labels_copy": (_int, [_vp, _vp, _vp]),
    "gee_io_labels_free": (None, [_vp]),
    "gee_io_labels_write": (_int, [_cs, _vp, _i64, _int]),
    "gee_io_csr_header": (_int, [_cs, _P_int, _P_i64, _P_i64]),
    "gee_io_csr_read": (_int, [_cs, _i64, _i64, _vp, _vp, _vp, _vp, _int]),
    "gee_io_csr_write": (_int, [_cs, _int, _i64, _i64, _vp, _vp, _vp, _int]),
    "gee_io_emb_header": (_int, [_cs, _P_i64, _P_i64]),
    "gee_io_emb_read": (_int, [_cs, _i64, _i64, _vp, _int]),
    "gee_io_emb_write": (_int, [_cs, _vp, _int, _i64, _i64, _int, _int]),
    "gee_io_expand_rows": (_int, [_vp, _vp, _vp, _i64, _i32, _vp, _int]),
}


def _load():
    if not os.path.exists(IO_LIB_PATH):
        raise ImportError(f"{IO_LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(IO_LIB_PATH)
    for name, (res, args) in IO_SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_io = None


def io_lib():
    global _io
    if _io is None:
        _io = _load()
    return _io


def _check(rc, path):
    if rc == GEE_IO_OK:
        return
    lib = io_lib()
    if rc == GEE_IO_ERR_OS:
        err = lib.gee_io_last_errno()
        raise OSError(err, os.strerror(err), str(path))
    msg = lib.gee_io_last_error().decode("utf-8", "replace")
    raise {GEE_IO_ERR_PARSE: ParseError, GEE_IO_ERR_FORMAT: FormatError,
           GEE_IO_ERR_VALUE: ValidationError}.get(rc, GeeError)(msg)


def _path(path):
    return os.fsencode(str(path))


def _threads(threads):
    return 0 if threads is None else int(threads)


def _p(a):
    if a is None:
        return None
    if _is_torch(a):
        return ctypes.c_void_p(a.data_ptr())
    return a.ctypes.data_as(ctypes.c_void_p)


def _host(a, dtype):
    """Host numpy view of an array or tensor (device tensors are copied down)."""
    if a is None:
        return None
    if _is_torch(a):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(a, dtype=dtype)


def _alloc(shape, dtype, pinned):
    if pinned:
        import torch

        t = torch.empty(shape, dtype={np.int64: torch.int64, np.int32: torch.int32, np.float32: torch.float32,
                                      np.float64: torch.float64}[dtype], pin_memory=True)
        return t
    return np.empty(shape, dtype=dtype)


# ------------------------------------------------------------- edge lists
def load_edge_list(path, weighted=False, directed=True, *, threads=None, device=None) -> EdgeList:
    """Parse a whitespace-separated text edge list (graph.py:94-145).

    Each line is ``u v`` or ``u v w``; lines starting with '#' are comments
    and blank lines are skipped.  Node ids are kept verbatim and
    ``n = 1 + max id``; an empty file yields the empty graph.  Raises
    ParseError naming the line number of the first malformed line.
    ``device`` (e.g. "cuda:0") returns the edge list on that GPU.
    """
    lib = io_lib()
    h = ctypes.c_void_p()
    _check(lib.gee_io_edges_parse(_path(path), int(bool(weighted)), _threads(threads), ctypes.byref(h)), path)
    try:
        s = lib.gee_io_edges_count(h)
        max_id = lib.gee_io_edges_max_id(h)
        if max_id + 1 > MAX_NODES:
            raise ValidationError(f"node count {max_id + 1} exceeds int32 limit {MAX_NODES}")
        pinned = device is not None
        src = _alloc(s, np.int32, pinned)
        dst = _alloc(s, np.int32, pinned)
        w = _alloc(s, np.float32, pinned) if weighted else None
        _check(lib.gee_io_edges_copy_i32(h, _p(src), _p(dst), _p(w), _threads(threads)), path)
    finally:
        lib.gee_io_edges_free(h)
    if device is not None:
        src, dst = src.to(device, non_blocking=True), dst.to(device, non_blocking=True)
        w = None if w is None else w.to(device, non_blocking=True)
    return EdgeList(n=max_id + 1, src=src, dst=dst, w=w, directed=directed)


def load_edge_list_f64(path, weighted=False, *, threads=None):
    """The parse in the reference's dtypes: (n, int64 src, int64 dst, f64 w)."""
    lib = io_lib()
    h = ctypes.c_void_p()
    _check(lib.gee_io_edges_parse(_path(path), int(bool(weighted)), _threads(threads), ctypes.byref(h)), path)
    try:
        s = lib.gee_io_edges_count(h)
        n = lib.gee_io_edges_max_id(h) + 1
        src, dst, w = np.empty(s, np.int64), np.empty(s, np.int64), np.empty(s, np.float64)
        _check(lib.gee_io_edges_copy_i64(h, _p(src), _p(dst), _p(w), _threads(threads)), path)
    finally:
        lib.gee_io_edges_free(h)
    return n, src, dst, w


def write_edge_list(el: EdgeList, path, *, threads=None) -> None:
    """Write the text edge-list format (graph.py:148-156); weights are
    omitted when all are 1 and otherwise written as repr(float(w))."""
    src = _host(el.src, np.int32)
    dst = _host(el.dst, np.int32)
    w = _host(el.w, np.float32)
    if w is not None and bool(np.all(w == 1.0)):
        w = None
    _check(io_lib().gee_io_edges_write(_path(path), _p(src), _p(dst), _p(w), int(src.shape[0]), _threads(threads)),
           path)


# -------------------------------------------------------- GEECSR1 cache
def read_binary_cache(path, *, threads=None, device=None) -> CsrGraph:
    """Read a binary CSR cache (graph.py:218-235); f64 weights are narrowed
    to the edge pass's float32 while reading.  ``device`` stages the arrays
    through pinned host memory onto that GPU."""
    lib = io_lib()
    d, n, s = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib.gee_io_csr_header(_path(path), ctypes.byref(d), ctypes.byref(n), ctypes.byref(s)), path)
    n, s = n.value, s.value
    pinned = device is not None
    offsets = _alloc(n + 1, np.int64, pinned)
    targets = _alloc(s, np.int32, pinned)
    weights = _alloc(s, np.float32, pinned)
    _check(lib.gee_io_csr_read(_path(path), n, s, _p(offsets), _p(targets), _p(weights), None, _threads(threads)),
           path)
    if device is not None:
        offsets, targets, weights = (a.to(device, non_blocking=True) for a in (offsets, targets, weights))
    return CsrGraph(n=n, offsets=offsets, targets=targets, weights=weights, directed=bool(d.value))


def write_binary_cache(g: CsrGraph, path, *, threads=None) -> None:
    """Write the little-endian binary CSR cache, magic GEECSR1 (graph.py:204-215)."""
    offsets = _host(g.offsets, np.int64)
    targets = _host(g.targets, np.int32)
    w = _host(g.weights, np.float32)
    _check(io_lib().gee_io_csr_write(_path(path), int(bool(g.directed)), int(g.n), int(targets.shape[0]),
                                     _p(offsets), _p(targets), _p(w), _threads(threads)), path)


# ---------------------------------------------------------------- labels
def load_labels(path, n, k, *, threads=None) -> LabelVector:
    """Load labels from text, auto-detecting the per-file format
    (labeling.py:33-73): one label per line (line i labels node i; exactly
    n data lines) or ``node label`` pairs (unlisted nodes default to 0)."""
    lib = io_lib()
    h = ctypes.c_void_p()
    _check(lib.gee_io_labels_parse(_path(path), _threads(threads), ctypes.byref(h)), path)
    try:
        width = lib.gee_io_labels_width(h)
        rows = lib.gee_io_labels_rows(h)
        c0 = np.empty(rows, np.int64)
        c1 = np.empty(rows, np.int64) if width == 2 else None
        _check(lib.gee_io_labels_copy(h, _p(c0), _p(c1)), path)
    finally:
        lib.gee_io_labels_free(h)
    labels = np.zeros(n, dtype=np.int64)
    if width == 1:
        if rows != n:
            raise ValidationError(f"{path}: {rows} labels for {n} nodes")
        bad = np.nonzero((c0 < 0) | (c0 > k))[0]
        if bad.size:
            i = int(bad[0])
            raise ValidationError(f"label {int(c0[i])} at node {i} outside [0, {k}]")
        labels[:] = c0
    elif width == 2:
        bad_node = (c0 < 0) | (c0 >= n)
        bad = np.nonzero(bad_node | (c1 < 0) | (c1 > k))[0]
        if bad.size:
            i = int(bad[0])
            if bad_node[i]:
                raise ValidationError(f"{path}: node {int(c0[i])} outside [0, {n})")
            raise ValidationError(f"label {int(c1[i])} at node {int(c0[i])} outside [0, {k}]")
        labels[c0] = c1  # repeated nodes: the last pair wins, as in the reference's loop
    return LabelVector(labels=labels, k=k)


def write_labels(y: LabelVector, path, *, threads=None) -> None:
    """Write the one-label-per-line format (labeling.py:81-84)."""
    lab = _host(y.labels, np.int32)
    _check(io_lib().gee_io_labels_write(_path(path), _p(lab), int(lab.shape[0]), _threads(threads)), path)


# ------------------------------------------------------------- embeddings
def write_embedding(z, path, fmt="csv", *, threads=None) -> None:
    """Write Z as csv (round-trip-exact decimals) or the binary format
    (encoder.py:209-221).  float32 Z is written as its exact float64 value;
    CUDA tensors are copied to the host first."""
    if _is_torch(z):
        z = z.detach()
        if z.dtype not in (__import__("torch").float32, __import__("torch").float64):
            z = z.double()
        z = z.cpu().numpy()
    z = np.asarray(z)
    if z.dtype not in (np.float32, np.float64):
        z = z.astype(np.float64)
    z = np.ascontiguousarray(z)
    if z.ndim != 2:
        raise ValidationError("embedding must be a 2-d array")
    if fmt not in ("csv", "binary"):
        raise ValidationError(f"unknown embedding format {fmt!r}")
    _check(io_lib().gee_io_emb_write(_path(path), _p(z), int(z.dtype == np.float64), int(z.shape[0]),
                                     int(z.shape[1]), 0 if fmt == "csv" else 1, _threads(threads)), path)


def read_embedding(path, *, threads=None) -> np.ndarray:
    """Read a binary embedding file back into an (n, k) float64 array
    (encoder.py:224-237)."""
    lib = io_lib()
    n, k = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.gee_io_emb_header(_path(path), ctypes.byref(n), ctypes.byref(k)), path)
    z = np.empty((n.value, k.value), np.float64)
    _check(lib.gee_io_emb_read(_path(path), n.value, k.value, _p(z), _threads(threads)), path)
    return z
