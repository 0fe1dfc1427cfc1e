"""CPU oracle for the GEE edge pass -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package, and only as the checker or
the CPU baseline.  The product package (paper_2402_04403_b200) never
imports it.

Two independent restatements of the reference (/root/reference/pkg/src/gee):
  * gee_oracle.c (liboracle.so, built by the Makefile here): serial_pass,
    bincount/build_projection, build_csr, and the pthreads port of
    embed_parallel's zero wave + arc wave with the CAS f64 atomic add;
  * numpy_reference: np.add.at scatter, restating the reference's own
    independent test oracle (tests/conftest.py:7-20 there).
Pinned against the reference's known-answer tests and golden vectors
generated from the reference itself (tests/golden/).
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_lib = None


def build(force=False):
    src = os.path.join(HERE, "gee_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(src) > os.path.getmtime(LIB_PATH):
        subprocess.run(["make", "-B" if force else "-s", "liboracle.so"], cwd=HERE, check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.oracle_bincount.argtypes = [vp, i64, i64, vp]
        L.oracle_bincount.restype = i32
        L.oracle_build_projection.argtypes = [vp, i64, i64, vp, vp, vp]
        L.oracle_build_projection.restype = i32
        L.oracle_serial_pass.argtypes = [vp, vp, vp, i64, vp, vp, vp, i64]
        L.oracle_serial_pass.restype = None
        L.oracle_build_csr.argtypes = [vp, vp, vp, i64, i64, i32, vp, vp, vp]
        L.oracle_build_csr.restype = None
        L.oracle_embed_parallel.argtypes = [vp, vp, vp, i32, vp, vp, vp, i64, i64, i32, i32, i32]
        L.oracle_embed_parallel.restype = None
        L.oracle_atomic_hammer.argtypes = [vp, i64, i64, dbl, i32]
        L.oracle_atomic_hammer.restype = None
        L.oracle_sampled_rows.argtypes = [vp, vp, vp, i64, vp, vp, vp, vp, i64]
        L.oracle_sampled_rows.restype = None
        u64 = ctypes.c_uint64
        L.oracle_sampled_rows_par.argtypes = [vp, vp, vp, i64, vp, vp, vp, vp, i64, vp, vp, i64, i32]
        L.oracle_sampled_rows_par.restype = None
        L.oracle_rmat.argtypes = [vp, vp, vp, i64, i64, i32, dbl, dbl, dbl, u64, i32, i32]
        L.oracle_rmat.restype = None
        L.oracle_uniform_labels.argtypes = [vp, i64, i64, u64]
        L.oracle_uniform_labels.restype = None
        L.oracle_build_csr_directed_par.argtypes = [vp, vp, vp, i64, i64, vp, vp, vp, i32]
        L.oracle_build_csr_directed_par.restype = None
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def bincount(labels, k):
    """np.bincount(labels, minlength=k+1) (encoder.py:87)."""
    lab = np.ascontiguousarray(labels, dtype=np.int64)
    counts = np.zeros(k + 1, dtype=np.int64)
    if lib().oracle_bincount(_p(lab), lab.size, k, _p(counts)):
        raise ValueError("label outside [0, k]")
    return counts


def projection(labels, k):
    """build_projection (encoder.py:80-103) -> (counts, inv f64[k+1], row_value f64[n])."""
    lab = np.ascontiguousarray(labels, dtype=np.int64)
    counts = np.zeros(k + 1, dtype=np.int64)
    inv = np.zeros(k + 1, dtype=np.float64)
    row = np.zeros(lab.size, dtype=np.float64)
    if lib().oracle_build_projection(_p(lab), lab.size, k, _p(counts), _p(inv), _p(row)):
        raise ValueError("label outside [0, k]")
    return counts, inv, row


def serial_embed(src, dst, w, labels, n, k):
    """embed_serial (encoder.py:106-120): f64 Z, both updates per listed edge,
    in list order.  w=None means unit weights."""
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    w = np.ones(src.size) if w is None else np.ascontiguousarray(w, dtype=np.float64)
    lab = np.ascontiguousarray(labels, dtype=np.int64)
    _, _, row = projection(lab, k)
    z = np.zeros((n, k), dtype=np.float64)
    if src.size:
        lib().oracle_serial_pass(_p(src), _p(dst), _p(w), src.size, _p(lab), _p(row), _p(z), k)
    return z


def build_csr(src, dst, w, n, directed):
    """build_csr (graph.py:159-184) -> (offsets int64, targets int32, weights f64)."""
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    w = np.ones(src.size) if w is None else np.ascontiguousarray(w, dtype=np.float64)
    arcs = src.size * (1 if directed else 2)
    offsets = np.zeros(n + 1, dtype=np.int64)
    targets = np.zeros(arcs, dtype=np.int32)
    weights = np.zeros(arcs, dtype=np.float64)
    lib().oracle_build_csr(_p(src), _p(dst), _p(w), src.size, n, 1 if directed else 0, _p(offsets),
                           _p(targets), _p(weights))
    return offsets, targets, weights


def parallel_embed(offsets, targets, weights, labels, k, directed, workers, atomics=True, out=None,
                   row_value=None, label32=None):
    """embed_parallel (encoder.py:123-194): pthreads port with the CAS f64
    atomic add; returns f64 Z (order-dependent rounding, like the reference)."""
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    targets = np.ascontiguousarray(targets, dtype=np.int32)
    n = offsets.size - 1
    unit = weights is None
    wts = np.zeros(1) if unit else np.ascontiguousarray(weights, dtype=np.float64)
    if row_value is None or label32 is None:
        _, _, row_value = projection(labels, k)
        label32 = np.ascontiguousarray(labels, dtype=np.int32)
    z = out if out is not None else np.empty((n, k), dtype=np.float64)
    lib().oracle_embed_parallel(_p(offsets), _p(targets), _p(wts), 1 if unit else 0, _p(label32), _p(row_value),
                                _p(z), n, k, 1 if directed else 0, 1 if atomics else 0, workers)
    return z


def atomic_hammer(reps, delta, threads):
    """atomic_add_hammer test hook (_kernels.py:109-114) on z[1]."""
    z = np.zeros(2)
    lib().oracle_atomic_hammer(_p(z), 1, reps, delta, threads)
    return z


def sampled_rows(src, dst, w, labels, k, rows):
    """f64 oracle rows Z[rows, :] by streaming the listed edges (serial_pass
    rule restricted to a row sample; for graphs whose full f64 Z does not fit
    in host memory)."""
    src = np.ascontiguousarray(src, dtype=np.int32)
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float32)
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    _, inv, _ = projection(lab, k)
    rows = np.asarray(rows, dtype=np.int64)
    slot = np.full(lab.size, -1, dtype=np.int64)
    slot[rows] = np.arange(rows.size)
    zs = np.zeros((rows.size, k), dtype=np.float64)
    lib().oracle_sampled_rows(_p(src), _p(dst), None if w is None else _p(w), src.size, _p(lab), _p(inv), _p(slot),
                              _p(zs), k)
    return zs


def sampled_rows_par(src, dst, w, labels, k, rows, threads=None):
    """sampled_rows over all host threads, plus the column mass: returns
    (zs f64[len(rows), k], mass f64[k]) with mass[c-1] = sum_x Z[x, c].
    For the full-size configurations (up to 1.8e9 listed edges)."""
    src = np.ascontiguousarray(src, dtype=np.int32)
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float32)
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    n = lab.size
    _, inv, _ = projection(lab, k)
    rows = np.asarray(rows, dtype=np.int64)
    assert np.unique(rows).size == rows.size, "rows must be distinct"
    keep = np.zeros((n + 63) // 64, dtype=np.uint64)
    np.bitwise_or.at(keep, rows >> 6, np.left_shift(np.uint64(1), (rows & 63).astype(np.uint64)))
    slot = np.zeros(n, dtype=np.int32)
    slot[rows] = np.arange(rows.size, dtype=np.int32)
    zs = np.empty((rows.size, k), dtype=np.float64)
    mass = np.empty(k + 1, dtype=np.float64)
    lib().oracle_sampled_rows_par(_p(src), _p(dst), None if w is None else _p(w), src.size, _p(lab), _p(inv),
                                  _p(keep), _p(slot), rows.size, _p(zs), _p(mass), k,
                                  threads or os.cpu_count() or 1)
    return zs, mass[1:]


def numpy_reference(src, dst, w, labels, n, k):
    """Vectorised np.add.at oracle, independent of the C restatement
    (restates the reference's tests/conftest.py:7-20)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    w = np.ones(src.size) if w is None else np.asarray(w, dtype=np.float64)
    lab = np.asarray(labels, dtype=np.int64)
    counts = np.bincount(lab, minlength=k + 1)
    inv = np.zeros(k + 1)
    nz = counts[1:] > 0
    inv[1:][nz] = 1.0 / counts[1:][nz]
    wrow = inv[lab]
    z = np.zeros((n, k))
    ys, yd = lab[src], lab[dst]
    m = yd > 0
    np.add.at(z, (src[m], yd[m] - 1), wrow[dst[m]] * w[m])
    m = ys > 0
    np.add.at(z, (dst[m], ys[m] - 1), wrow[src[m]] * w[m])
    return z


# ------------------------------------------------ CPU arm inputs (bench.py)
RMAT_ABC = (0.57, 0.19, 0.19)


def rmat_edges(scale, s, seed, weighted=False, first=0, threads=None, scramble=True):
    """C restatement of synth.rmat_edges_numpy: int32 src/dst (+ f32 w), all
    host threads.  The reference arm builds its inputs with this, so it never
    loads the product library."""
    src = np.empty(s, dtype=np.int32)
    dst = np.empty(s, dtype=np.int32)
    w = np.empty(s, dtype=np.float32) if weighted else None
    a, b, c = RMAT_ABC
    lib().oracle_rmat(_p(src), _p(dst), None if w is None else _p(w), first, s, scale, a, b, c,
                      seed & ((1 << 64) - 1), 1 if scramble else 0, threads or os.cpu_count() or 1)
    return src, dst, w


def uniform_labels(n, k, seed):
    """C restatement of synth.uniform_labels_numpy (int32, 1..k)."""
    y = np.empty(n, dtype=np.int32)
    lib().oracle_uniform_labels(_p(y), n, k, seed & ((1 << 64) - 1))
    return y


def build_csr_directed_par(src, dst, w, n, threads=None):
    """Directed build_csr (graph.py:159-184) in the reference dtypes (int64
    offsets, int32 targets, f64 weights or None for unit), threaded; arc
    order within a row unspecified."""
    src = np.ascontiguousarray(src, dtype=np.int32)
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    s = src.size
    offsets = np.empty(n + 1, dtype=np.int64)
    targets = np.empty(s, dtype=np.int32)
    weights = np.empty(s, dtype=np.float64) if w is not None else None
    wf = None if w is None else np.ascontiguousarray(w, dtype=np.float32)
    lib().oracle_build_csr_directed_par(_p(src), _p(dst), None if wf is None else _p(wf), s, n, _p(offsets),
                                        _p(targets), None if weights is None else _p(weights),
                                        threads or os.cpu_count() or 1)
    return offsets, targets, weights
