"""Throughput of the native data formats (libgee_io.so) vs the reference's readers.

    python tools/io_bench.py [--edges 32000000] [--ref-edges 2000000] [--out profiles/io_bench.json]

Text edge list (C2-shaped: weighted, n = 1e6), label file, GEECSR1 cache
and GEEEMB1 / csv embedding: ours on every host thread, and -- when
/root/reference is present (build container only) -- the reference's own
functions on a bounded sample, reported per line / per byte.  Files live in
a temp dir (page cache warm after the write, as for a re-read of a cache).
"""

import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2402_04403_b200 as gb  # noqa: E402
from paper_2402_04403_b200 import formats  # noqa: E402


def timed(fn, reps=3):
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--edges", type=int, default=32_000_000)
    ap.add_argument("--nodes", type=int, default=1_000_000)
    ap.add_argument("--ref-edges", type=int, default=2_000_000)
    ap.add_argument("--emb-rows", type=int, default=200_000)
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rng = np.random.default_rng(1)
    tmp = tempfile.mkdtemp(prefix="gee_iobench_")
    res = {"host_threads": os.cpu_count(), "edges": args.edges, "nodes": args.nodes}

    s, n = args.edges, args.nodes
    el = gb.EdgeList(n=n, src=rng.integers(0, n, s), dst=rng.integers(0, n, s),
                     w=(1 - rng.random(s)).astype(np.float32))
    txt = os.path.join(tmp, "g.txt")
    t, _ = timed(lambda: gb.write_edge_list(el, txt), reps=1)
    size = os.path.getsize(txt)
    res["text_bytes"] = size
    res["write_edge_list_s"] = t
    t, got = timed(lambda: gb.load_edge_list(txt, weighted=True))
    assert got.s == s
    res["load_edge_list_s"] = t
    res["load_edge_list_medges_per_s"] = s / t / 1e6
    res["load_edge_list_mb_per_s"] = size / t / 1e6

    g = gb.CsrGraph(n=n, offsets=np.concatenate([[0], np.cumsum(np.bincount(el.src, minlength=n))]),
                    targets=el.dst[np.argsort(el.src, kind="stable")],
                    weights=el.w[np.argsort(el.src, kind="stable")])
    cache = os.path.join(tmp, "g.bin")
    t, _ = timed(lambda: gb.write_binary_cache(g, cache), reps=1)
    res["write_binary_cache_gb_per_s"] = os.path.getsize(cache) / t / 1e9
    t, _ = timed(lambda: gb.read_binary_cache(cache))
    res["read_binary_cache_gb_per_s"] = os.path.getsize(cache) / t / 1e9

    lab = rng.integers(0, 51, n).astype(np.int32)
    lp = os.path.join(tmp, "y.txt")
    gb.write_labels(gb.LabelVector(labels=lab, k=50), lp)
    t, _ = timed(lambda: gb.load_labels(lp, n, 50))
    res["load_labels_mlines_per_s"] = n / t / 1e6

    z = np.zeros((args.emb_rows, args.k), np.float32)
    nz = rng.random(z.shape) < 0.3
    z[nz] = rng.random(int(nz.sum())).astype(np.float32)
    for fmt in ("binary", "csv"):
        p = os.path.join(tmp, f"z.{fmt}")
        t, _ = timed(lambda: gb.write_embedding(z, p, fmt=fmt), reps=1)
        res[f"write_embedding_{fmt}_mvalues_per_s"] = z.size / t / 1e6

    if os.path.isdir("/root/reference/pkg/src/gee"):
        sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
        from make_golden import import_reference

        ref = import_reference()
        m = min(args.ref_edges, s)
        with open(txt, "rb") as fh:
            head = b"".join(fh.readline() for _ in range(m))
        sp = os.path.join(tmp, "sample.txt")
        open(sp, "wb").write(head)
        t, rel = timed(lambda: ref.load_edge_list(sp, weighted=True), reps=1)
        res["reference_load_edge_list_medges_per_s"] = m / t / 1e6
        t, _ = timed(lambda: gb.load_edge_list(sp, weighted=True))
        res["sample_load_edge_list_medges_per_s"] = m / t / 1e6
        rg = ref.CsrGraph(n=g.n, offsets=g.offsets, targets=g.targets, weights=g.weights.astype(np.float64))
        t, _ = timed(lambda: ref.write_binary_cache(rg, cache), reps=1)
        res["reference_write_binary_cache_gb_per_s"] = os.path.getsize(cache) / t / 1e9
        t, _ = timed(lambda: ref.read_binary_cache(cache), reps=1)
        res["reference_read_binary_cache_gb_per_s"] = os.path.getsize(cache) / t / 1e9
        t, _ = timed(lambda: ref.load_labels(lp, n, 50), reps=1)
        res["reference_load_labels_mlines_per_s"] = n / t / 1e6
        zs = z[:20_000].astype(np.float64)
        for fmt in ("binary", "csv"):
            p = os.path.join(tmp, f"rz.{fmt}")
            t, _ = timed(lambda: ref.write_embedding(zs, p, fmt=fmt), reps=1)
            res[f"reference_write_embedding_{fmt}_mvalues_per_s"] = zs.size / t / 1e6
    line = json.dumps(res)
    print(line)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(line + "\n")
    for f in os.listdir(tmp):
        os.unlink(os.path.join(tmp, f))
    os.rmdir(tmp)


if __name__ == "__main__":
    main()
