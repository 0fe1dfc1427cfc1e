"""Whole-call time of embed_parallel / embed_serial per variant vs graph size
(the measured table behind encoder.PUSH_MAX_ARCS).

Host arrays in, host Z out, as the reference's API is called; wall clock,
median of 5 after a warm-up.  Usage: python tools/variant_table.py OUT.json
"""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2402_04403_b200 as gb  # noqa: E402


def timed(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def main(out):
    rows = []
    rng = np.random.default_rng(1)
    for s in (10_000, 30_000, 100_000, 300_000, 1_000_000, 3_000_000, 10_000_000, 30_000_000):
        n = max(16, s // 16)
        src = rng.integers(0, n, s).astype(np.int32)
        dst = rng.integers(0, n, s).astype(np.int32)
        w = (1.0 - rng.random(s)).astype(np.float32)
        y = gb.random_labels(n, 50, 1.0, seed=s)
        el = gb.EdgeList(n=n, src=src, dst=dst, w=w, directed=False)
        g = gb.build_csr(el)
        row = {"s": s, "n": n, "arcs": int(g.targets.shape[0]), "k": 50}
        for v in ("pull", "push"):
            row[f"parallel_{v}_ms"] = 1e3 * timed(lambda: gb.embed_parallel(g, y, variant=v))
            row[f"serial_{v}_ms"] = 1e3 * timed(lambda: gb.embed_serial(el, y, variant=v))
        rows.append(row)
        print(json.dumps(row), flush=True)
    with open(out, "w") as f:
        json.dump({"what": "whole-call wall time (host arrays in, host Z out), median of 5", "rows": rows}, f,
                  indent=1)


if __name__ == "__main__":
    main(sys.argv[1])
