"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference datasets (SNAP, Friendster) are not available; seeded
synthetic graphs with the configurations' shapes stand in for them
(SURVEY.md section 8d).  R-MAT / ER / uniform labels come from the
counter-based generator in csrc/gee_synth.cu (GPU, any slice
independently); SBM graphs and random_labels use numpy default_rng as the
reference does (graph.py:198, labeling.py:100).  `*_numpy` functions
restate the GPU streams exactly for tests.
"""

from dataclasses import dataclass

import numpy as np

from .errors import ValidationError

M64 = (1 << 64) - 1

RMAT_ABC = (0.57, 0.19, 0.19)  # d = 0.05


# ------------------------------------------------------------ GPU streams
def _lib():
    from . import _lib as L

    return L


def rmat_edges(scale, s, seed, weighted=False, a=RMAT_ABC[0], b=RMAT_ABC[1], c=RMAT_ABC[2], scramble=True,
               first=0, device=None, out=None):
    """R-MAT edges [first, first+s) as CUDA int32 src/dst (+ fp32 w)."""
    import torch

    from .device import require_cuda

    L = _lib()
    dev = require_cuda(device)
    if out is None:
        src = torch.empty(s, dtype=torch.int32, device=dev)
        dst = torch.empty(s, dtype=torch.int32, device=dev)
        w = torch.empty(s, dtype=torch.float32, device=dev) if weighted else None
    else:
        src, dst, w = out
    L.check(L.lib.gee_synth_rmat(L.ptr(src), L.ptr(dst), L.ptr(w), first, s, scale, a, b, c, seed & M64,
                                 1 if scramble else 0, L.stream_handle()), "gee_synth_rmat")
    return src, dst, w


def er_edges(n, s, seed, weighted=False, first=0, device=None):
    """G(n, s) edges [first, first+s) (with replacement) as CUDA arrays."""
    import torch

    from .device import require_cuda

    L = _lib()
    dev = require_cuda(device)
    src = torch.empty(s, dtype=torch.int32, device=dev)
    dst = torch.empty(s, dtype=torch.int32, device=dev)
    w = torch.empty(s, dtype=torch.float32, device=dev) if weighted else None
    L.check(L.lib.gee_synth_er(L.ptr(src), L.ptr(dst), L.ptr(w), first, s, n, seed & M64, L.stream_handle()),
            "gee_synth_er")
    return src, dst, w


def uniform_labels(n, k, seed, device=None):
    import torch

    from .device import require_cuda

    L = _lib()
    dev = require_cuda(device)
    y = torch.empty(n, dtype=torch.int32, device=dev)
    L.check(L.lib.gee_synth_uniform_labels(L.ptr(y), n, k, seed & M64, L.stream_handle()),
            "gee_synth_uniform_labels")
    return y


# ------------------------------------------------- numpy restatements
def _splitmix64(x):
    x = (x + np.uint64(0x9E3779B97F4A7C15)) & np.uint64(M64)
    x = ((x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & np.uint64(M64)
    x = ((x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & np.uint64(M64)
    return x ^ (x >> np.uint64(31))


def word_numpy(seed, tag, ctr):
    """gee_synth_word for a vector of counters."""
    with np.errstate(over="ignore"):
        key = _splitmix64(np.uint64(seed & M64) ^ np.uint64((tag * 0xD1B54A32D192ED03) & M64))
        return _splitmix64((key + np.asarray(ctr, dtype=np.uint64)) & np.uint64(M64))


def _scramble_numpy(x, scale, m1, m2):
    mask = np.uint64((1 << scale) - 1)
    h = max(scale // 2, 1)
    with np.errstate(over="ignore"):
        x = (x * np.uint64(m1)) & mask
        x ^= x >> np.uint64(h)
        x = (x * np.uint64(m2)) & mask
        x ^= x >> np.uint64(h + (scale & 1))
        x = (x * np.uint64(m1)) & mask
    return x


def rmat_edges_numpy(scale, s, seed, weighted=False, a=RMAT_ABC[0], b=RMAT_ABC[1], c=RMAT_ABC[2],
                     scramble=True, first=0):
    """Exact numpy restatement of gee_synth_rmat (small s only)."""
    two32 = 4294967296.0
    ta, tab, tabc = np.uint64(int(a * two32)), np.uint64(int((a + b) * two32)), np.uint64(int((a + b + c) * two32))
    i = np.arange(first, first + s, dtype=np.uint64)
    u = np.zeros(s, dtype=np.uint64)
    v = np.zeros(s, dtype=np.uint64)
    bits = None
    for lvl in range(scale):
        if lvl % 2 == 0:
            with np.errstate(over="ignore"):
                bits = word_numpy(seed, 1, i * np.uint64(32) + np.uint64(lvl >> 1))
        r = (bits >> np.uint64(32)) if lvl % 2 else (bits & np.uint64(0xFFFFFFFF))
        bu = (r >= tab).astype(np.uint64)
        bv = (((r >= ta) & (r < tab)) | (r >= tabc)).astype(np.uint64)
        u = (u << np.uint64(1)) | bu
        v = (v << np.uint64(1)) | bv
    if scramble:
        with np.errstate(over="ignore"):
            m1 = int(_splitmix64(np.uint64(seed & M64) ^ np.uint64(0x5EED1))) | 1
            m2 = int(_splitmix64(np.uint64(seed & M64) ^ np.uint64(0x5EED2))) | 1
        u = _scramble_numpy(u, scale, m1, m2)
        v = _scramble_numpy(v, scale, m1, m2)
    w = None
    if weighted:
        w = (1.0 - (word_numpy(seed, 2, i) >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)
             ).astype(np.float32)
    return u.astype(np.int32), v.astype(np.int32), w


def er_edges_numpy(n, s, seed, weighted=False, first=0):
    i = np.arange(first, first + s, dtype=np.uint64)
    r = word_numpy(seed, 3, i)
    src = (((r & np.uint64(0xFFFFFFFF)) * np.uint64(n)) >> np.uint64(32)).astype(np.int32)
    dst = (((r >> np.uint64(32)) * np.uint64(n)) >> np.uint64(32)).astype(np.int32)
    w = None
    if weighted:
        w = (1.0 - (word_numpy(seed, 2, i) >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)
             ).astype(np.float32)
    return src, dst, w


def uniform_labels_numpy(n, k, seed):
    r = word_numpy(seed, 4, np.arange(n, dtype=np.uint64)) >> np.uint64(32)
    return (1 + ((r * np.uint64(k)) >> np.uint64(32))).astype(np.int32)


# ------------------------------------------------------- numpy-only inputs
def sbm_undirected(n, k, p_in, p_out, seed):
    """C1: labels iid uniform {1..k}; each pair i<j an edge w.p. p_in (same
    block) or p_out.  Returns (src, dst, labels) int32; each edge listed once."""
    rng = np.random.default_rng(seed)
    y = rng.integers(1, k + 1, size=n, dtype=np.int64)
    src_parts, dst_parts = [], []
    for i in range(n - 1):
        j = np.arange(i + 1, n)
        p = np.where(y[j] == y[i], p_in, p_out)
        hit = j[rng.random(j.size) < p]
        src_parts.append(np.full(hit.size, i, dtype=np.int64))
        dst_parts.append(hit)
    src = np.concatenate(src_parts) if src_parts else np.zeros(0, np.int64)
    dst = np.concatenate(dst_parts) if dst_parts else np.zeros(0, np.int64)
    return src.astype(np.int32), dst.astype(np.int32), y.astype(np.int32)


def sbm_directed(n, k, s, p_same, seed):
    """C2: labels iid uniform {1..k}; src uniform; dst drawn from src's block
    w.p. p_same, else uniform; fp32 weights 1 - U[0,1) in (0, 1]."""
    rng = np.random.default_rng(seed)
    y = rng.integers(1, k + 1, size=n, dtype=np.int64)
    order = np.argsort(y, kind="stable")
    starts = np.searchsorted(y[order], np.arange(1, k + 2))
    src = rng.integers(0, n, size=s, dtype=np.int64)
    dst = rng.integers(0, n, size=s, dtype=np.int64)
    same = rng.random(s) < p_same
    cls = y[src[same]]
    lo, hi = starts[cls - 1], starts[cls]
    pick = lo + (rng.random(cls.size) * (hi - lo)).astype(np.int64)
    dst[same] = order[np.minimum(pick, hi - 1)]
    w = (1.0 - rng.random(s, dtype=np.float32)).astype(np.float32)
    return src.astype(np.int32), dst.astype(np.int32), w, y.astype(np.int32)


def zipf_labels(n, k, s_exp, seed):
    """C5: every node labeled; class sizes n_c = round(n c^-s / H) with the
    largest-remainder rule, assigned over a seeded permutation."""
    c = np.arange(1, k + 1, dtype=np.float64)
    share = c ** (-s_exp)
    share /= share.sum()
    exact = n * share
    sizes = np.floor(exact).astype(np.int64)
    short = n - int(sizes.sum())
    if short:
        sizes[np.argsort(-(exact - sizes), kind="stable")[:short]] += 1
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    y = np.empty(n, dtype=np.int32)
    y[perm] = np.repeat(np.arange(1, k + 1, dtype=np.int32), sizes)
    return y


# ------------------------------------------------------------ configs
@dataclass
class Config:
    name: str
    n: int
    s: int
    k: int
    weighted: bool
    directed: bool
    note: str


CONFIGS = {
    1: Config("C1-sbm-n1e4-k5", 10_000, 0, 5, False, False,
              "SBM p_in=0.01 p_out=0.001, undirected, unit weights, all labeled (seed 0)"),
    2: Config("C2-sbm-n1e6-k50", 1_000_000, 32_000_000, 50, True, True,
              "directed SBM, out-degree 32, p_same=0.5, fp32 w in (0,1], all labeled (seed 2)"),
    3: Config("C3-rmat-s24-k100", 1 << 24, (1 << 24) * 16, 100, False, False,
              "R-MAT(.57,.19,.19,.05) scale 24 ef 16, undirected, unit, 10% labeled (seed 3)"),
    4: Config("C4-rmat-s27-k50", 1 << 27, 1_800_000_000, 50, True, True,
              "R-MAT(.57,.19,.19,.05) scale 27, 1.8e9 directed edges, fp32 w in (0,1], all labeled (seed 4)"),
    5: Config("C5-er-n4e6-k1000", 4_000_000, 256_000_000, 1000, False, False,
              "ER G(n,s) n=4e6 s=2.56e8, undirected, unit, Zipf(1.1) labels (seed 5)"),
}


def make_config(idx, device=None, scale_override=None, edges_override=None):
    """Generate config `idx` on the GPU: returns (src, dst, w, labels, n, k, directed)
    as CUDA tensors (w None for unit weights).  scale_override / edges_override
    shrink R-MAT / ER configs for tests."""
    import torch

    from .device import require_cuda, to_device

    dev = require_cuda(device)
    cfg = CONFIGS[idx]
    if idx == 1:
        src, dst, y = sbm_undirected(cfg.n, cfg.k, 0.01, 0.001, seed=0)
        return (to_device(src, torch.int32, dev), to_device(dst, torch.int32, dev), None,
                to_device(y, torch.int32, dev), cfg.n, cfg.k, False)
    if idx == 2:
        n, s = cfg.n, cfg.s
        if edges_override:
            s = edges_override
        src, dst, w, y = sbm_directed(n, cfg.k, s, 0.5, seed=2)
        return (to_device(src, torch.int32, dev), to_device(dst, torch.int32, dev), to_device(w, torch.float32, dev),
                to_device(y, torch.int32, dev), n, cfg.k, True)
    if idx in (3, 4):
        scale = 24 if idx == 3 else 27
        ef_s = cfg.s
        if scale_override:
            ef_s = int(round(cfg.s / cfg.n * (1 << scale_override)))
            scale = scale_override
        if edges_override:
            ef_s = edges_override
        n = 1 << scale
        src, dst, w = rmat_edges(scale, ef_s, seed=idx, weighted=cfg.weighted, device=dev)
        if idx == 3:
            from .labeling import random_labels

            y = to_device(random_labels(n, cfg.k, 0.1, seed=3).labels, torch.int32, dev)
        else:
            y = uniform_labels(n, cfg.k, seed=4, device=dev)
        return src, dst, w, y, n, cfg.k, cfg.directed
    if idx == 5:
        n, s = cfg.n, cfg.s
        if edges_override:
            s = edges_override
            n = max(1, int(round(cfg.n * s / cfg.s)))
        src, dst, _ = er_edges(n, s, seed=5, device=dev)
        y = to_device(zipf_labels(n, cfg.k, 1.1, seed=5), torch.int32, dev)
        return src, dst, None, y, n, cfg.k, False
    raise ValidationError(f"unknown config {idx}")
