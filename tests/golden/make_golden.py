"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg/src/gee to a temp dir (numba must not write
caches into the read-only reference tree), imports it, and records inputs
and outputs of build_projection / class_counts / build_csr / embed_serial /
embed_parallel on seeded inputs into tests/golden/golden.npz.  The GPU box
never reads /root/reference; tests only read the committed .npz.
"""

import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src/gee"


def import_reference():
    tmp = tempfile.mkdtemp(prefix="gee_ref_")
    shutil.copytree(REF, os.path.join(tmp, "gee"))
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tmp, "numba_cache"))
    sys.path.insert(0, tmp)
    import gee  # noqa: E402

    return gee


def main():
    gee = import_reference()
    out = {}
    rng = np.random.default_rng(20240811)  # the reference's conftest seed

    def add_case(name, el, y, workers=4):
        out[f"{name}/n"] = np.int64(el.n)
        out[f"{name}/k"] = np.int64(y.k)
        out[f"{name}/directed"] = np.int64(el.directed)
        out[f"{name}/src"] = el.src.astype(np.int64)
        out[f"{name}/dst"] = el.dst.astype(np.int64)
        out[f"{name}/w"] = el.w.astype(np.float64)
        out[f"{name}/labels"] = y.labels.astype(np.int64)
        proj = gee.build_projection(y)
        out[f"{name}/row_value"] = proj.row_value
        out[f"{name}/class_counts"] = gee.class_counts(y).astype(np.int64)
        out[f"{name}/z_serial"] = gee.embed_serial(el, y)
        g = gee.build_csr(el)
        out[f"{name}/csr_offsets"] = g.offsets
        out[f"{name}/csr_targets"] = g.targets
        out[f"{name}/csr_weights"] = g.weights
        out[f"{name}/z_parallel"] = gee.embed_parallel(g, y, workers=workers)

    # known-answer cases from the reference tests
    add_case("chain", gee.EdgeList(n=3, src=[0, 1], dst=[1, 2], w=[1.0, 1.0], directed=True),
             gee.LabelVector(labels=[1, 1, 2], k=2))
    add_case("mirror", gee.EdgeList(n=2, src=[0], dst=[1], w=[1.0], directed=False),
             gee.LabelVector(labels=[1, 2], k=2))
    leaves = 1000
    add_case("star", gee.EdgeList(n=leaves + 1, src=np.zeros(leaves, dtype=np.int64),
                                  dst=np.arange(1, leaves + 1, dtype=np.int64), w=np.ones(leaves), directed=False),
             gee.LabelVector(labels=[0] + [1] * leaves, k=1))
    hubs = 2000
    n = hubs + 2
    leaf_ids = np.arange(1, hubs + 1, dtype=np.int64)
    labels = np.zeros(n, dtype=np.int64)
    labels[0] = labels[n - 1] = 1
    add_case("two_hub", gee.EdgeList(n=n, src=np.concatenate([np.zeros(hubs, np.int64), np.full(hubs, n - 1)]),
                                     dst=np.concatenate([leaf_ids, leaf_ids]), w=np.ones(2 * hubs), directed=True),
             gee.LabelVector(labels=labels, k=2))
    add_case("self_loops", gee.EdgeList(n=4, src=[0, 0, 1, 2, 2], dst=[0, 1, 1, 3, 3], w=[1.0, 2.0, 0.5, 1.0, 1.0],
                                        directed=True),
             gee.LabelVector(labels=[1, 2, 0, 1], k=2))
    add_case("empty", gee.EdgeList(n=4, src=[], dst=[], w=[]), gee.LabelVector(labels=[1, 0, 2, 0], k=2))
    add_case("unlabeled", gee.EdgeList(n=3, src=[0, 1], dst=[1, 2], w=[2.0, 1.0]),
             gee.LabelVector(labels=[0, 0, 0], k=3))

    # random battery, the reference's generator shapes (conftest.py:23-39)
    for i in range(10):
        n = int(rng.integers(2, 2000))
        s = int(rng.integers(0, 20000))
        src = rng.integers(0, n, size=s, dtype=np.int64)
        dst = rng.integers(0, n, size=s, dtype=np.int64)
        if i % 3 == 0:
            w = np.ones(s)
        else:  # fp32-representable weights in (0, 2] so the GPU sees the same values
            w = (2.0 * (1.0 - rng.random(s))).astype(np.float32).astype(np.float64)
        el = gee.EdgeList(n=n, src=src, dst=dst, w=w, directed=bool(i % 2))
        k = int(rng.integers(1, 12))
        frac = [0.2, 1.0, 0.5][i % 3]
        y = gee.random_labels(n, k, frac, int(rng.integers(0, 2**31)))
        out[f"rand{i}/seed_note"] = np.int64(i)
        add_case(f"rand{i}", el, y)

    # projection-only KATs and random label vectors (class counts)
    for i, (labels, k) in enumerate([([1, 1, 2], 2), ([0, 0], 3), ([2], 2), ([1, 2, 2, 2, 2], 2),
                                     ([1, 1], 3), ([0, 0, 0], 2)]):
        y = gee.LabelVector(labels=labels, k=k)
        out[f"proj{i}/labels"] = y.labels
        out[f"proj{i}/k"] = np.int64(k)
        out[f"proj{i}/dense"] = gee.build_projection(y).to_dense()
        out[f"proj{i}/class_counts"] = gee.class_counts(y)
    for i in range(5):
        n = int(rng.integers(1, 50000))
        k = int(rng.integers(1, 300))
        y = gee.LabelVector(labels=rng.integers(0, k + 1, n), k=k)
        out[f"counts{i}/labels"] = y.labels
        out[f"counts{i}/k"] = np.int64(k)
        out[f"counts{i}/bincount"] = np.bincount(y.labels, minlength=k + 1)

    # random_labels stream: (n, k, fraction, seed) -> labels
    for i, (n, k, f, seed) in enumerate([(1003, 7, 0.25, 11), (50, 5, 0.4, 3), (100000, 50, 0.1, 9)]):
        out[f"rl{i}/args"] = np.array([n, k, seed], dtype=np.int64)
        out[f"rl{i}/fraction"] = np.float64(f)
        out[f"rl{i}/labels"] = gee.random_labels(n, k, f, seed).labels

    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
