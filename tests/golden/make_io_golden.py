"""Golden fixtures for the data formats, produced by the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_io_golden.py

For every case below it runs the reference's own reader or writer
(load_edge_list, load_labels, read_binary_cache / write_binary_cache,
read_embedding / write_embedding, write_edge_list, write_labels) and records
the outcome -- parsed arrays, written bytes, or the exception type and text
(with the file path replaced by "{path}") -- in tests/golden/io_cases.json.
tests/test_formats.py replays the same inputs through libgee_io.so.
"""

import base64
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import import_reference  # noqa: E402

# (name, file bytes, weighted) -- text edge lists, graph.py:94-145
EDGE_CASES = [
    ("comments_unit", b"# c\n0 1\n1 2\n", False),
    ("weighted", b"0 1 2.5\n", True),
    ("bad_id", b"0 x\n", False),
    ("negative_line2", b"0 1\n-1 2\n", False),
    ("inf_weight", b"0 1 inf\n", True),
    ("nan_weight", b"0 1 nan\n", True),
    ("neg_infinity_weight", b"0 1 -Infinity\n", True),
    ("overflow_weight", b"0 1 1e400\n", True),
    ("hex_weight", b"0 1 0x1p3\n", True),
    ("bad_exponent", b"0 1 1e\n", True),
    ("missing_weight", b"0 1\n", True),
    ("too_many", b"0 1 2 3\n", False),
    ("one_field", b"\n\n7\n", False),
    ("empty", b"", False),
    ("only_comments", b"# a\n#b\n\n", True),
    ("blank_tabs", b"\n3\t4\n  \n", False),
    ("verbatim_ids", b"7 9\n", False),
    ("crlf", b"0 1 0.25\r\n2 3 0.5\r\n\r\n4 5 1\r\n", True),
    ("cr_only", b"0 1\r1 2\r\r3 x\r", False),
    ("no_final_newline", b"0 1\n5 2", False),
    ("third_field_ignored", b"0 1 junk\n2 3 4\n", False),
    ("underscores", b"1_0 +2 1_0.5\n007 -0 .5\n3 4 5.\n", True),
    ("bad_underscore_id", b"1__0 2\n", False),
    ("bad_underscore_w", b"1 2 1._5\n", True),
    ("exp_underscore_w", b"1 2 1e1_0\n", True),
    ("hash_not_first", b"0 1\n  # not a comment\n", False),
    ("id_is_float", b"0 1.0\n", False),
    ("error_after_comments", b"# a\n\n0 1\n# b\n\n1 2 3 4\n", False),
    ("weights_many", b"0 1 1e-3\n1 2 0.1\n2 3 3.4028234663852886e38\n3 4 1e-45\n4 5 -2.5E+2\n5 6 123456789.123456789\n"
                     b"6 7 0.30000000000000004\n7 8 1E22\n8 9 9007199254740993\n", True),
    ("vtab_ff_ws", b"0\x0b1\n2\x0c3\n4\x1f5\n", False),
]

# (name, file bytes, n, k) -- label files, labeling.py:33-73
LABEL_CASES = [
    ("sequential", b"1\n0\n2\n", 3, 2),
    ("pairs_default_zero", b"0 1\n2 2\n", 4, 2),
    ("out_of_range", b"1\n3\n", 2, 2),
    ("negative_label", b"1\n-1\n", 2, 2),
    ("pair_node_out_of_range", b"0 1\n5 1\n", 3, 2),
    ("pair_node_negative", b"-1 1\n", 3, 2),
    ("pair_label_bad_before_node", b"0 9\n7 1\n", 3, 2),
    ("wrong_count", b"1\n1\n", 3, 2),
    ("mixed", b"1\n0 1\n", 2, 2),
    ("non_integer", b"1\nx\n", 2, 2),
    ("three_fields", b"# c\n1 2 3\n", 2, 2),
    ("comments", b"# header\n1\n\n# mid\n2\n", 2, 2),
    ("empty", b"", 3, 2),
    ("pairs_repeat_last_wins", b"1 1\n1 2\n", 2, 2),
    ("crlf_pairs", b"0 1\r\n1 2\r\n", 2, 2),
    ("k_zero", b"0\n0\n", 2, 0),
]


def b64(b):
    return base64.b64encode(b).decode("ascii")


def outcome(fn, path):
    try:
        return {"ok": fn()}
    except Exception as exc:  # record the reference's exception verbatim
        return {"error": type(exc).__name__, "message": str(exc).replace(str(path), "{path}")}


def main():
    gee = import_reference()
    tmp = tempfile.mkdtemp(prefix="gee_io_golden_")
    path = os.path.join(tmp, "f")
    out = {"edges": [], "labels": [], "csr": [], "emb": [], "write_edges": [], "write_labels": []}

    for name, data, weighted in EDGE_CASES:
        with open(path, "wb") as fh:
            fh.write(data)

        def run():
            el = gee.load_edge_list(path, weighted=weighted)
            return {"n": int(el.n), "src": el.src.tolist(), "dst": el.dst.tolist(), "w": [float(x) for x in el.w]}

        out["edges"].append({"name": name, "data": b64(data), "weighted": weighted, **outcome(run, path)})

    for name, data, n, k in LABEL_CASES:
        with open(path, "wb") as fh:
            fh.write(data)
        out["labels"].append({"name": name, "data": b64(data), "n": n, "k": k,
                              **outcome(lambda: gee.load_labels(path, n, k).labels.tolist(), path)})

    # GEECSR1: files written by the reference, and corrupted variants
    rng = np.random.default_rng(7)
    graphs = {
        "chain_directed": gee.EdgeList(n=3, src=[0, 1], dst=[1, 2], w=[1.0, 1.0], directed=True),
        "weighted_undirected": gee.EdgeList(n=6, src=[0, 1, 2, 5, 3], dst=[1, 2, 0, 5, 4],
                                            w=np.float32([0.5, 0.25, 1.5, 3.0, 0.1]).astype(np.float64),
                                            directed=False),
        "random": gee.EdgeList(n=40, src=rng.integers(0, 40, 300), dst=rng.integers(0, 40, 300),
                               w=rng.random(300).astype(np.float32).astype(np.float64), directed=True),
        "empty": gee.EdgeList(n=0, src=[], dst=[], w=[], directed=True),
        "isolated": gee.EdgeList(n=5, src=[], dst=[], w=[], directed=False),
    }
    for name, el in graphs.items():
        g = gee.build_csr(el)
        gee.write_binary_cache(g, path)
        data = open(path, "rb").read()
        out["csr"].append({"name": name, "data": b64(data), "n": int(g.n), "directed": bool(g.directed),
                           "offsets": g.offsets.tolist(), "targets": g.targets.tolist(),
                           "weights": [float(x) for x in g.weights]})
    good = b64(open(path, "rb").read())
    base = base64.b64decode(out["csr"][2]["data"])
    for name, data in [("bad_magic", b"NOTACSR\x00" + base[8:]), ("truncated_header", base[:20]),
                       ("bad_version", base[:8] + b"\x02" + base[9:]), ("short_payload", base[:-3]),
                       ("long_payload", base + b"\x00"), ("zero_bytes", b"")]:
        with open(path, "wb") as fh:
            fh.write(data)
        out["csr"].append({"name": name, "data": b64(data), **outcome(lambda: gee.read_binary_cache(path), path)})
    del good

    # GEEEMB1 / csv: what the reference writes for float32-valued Z
    tricky = np.float32([0.0, -0.0, 1.0, 1 / 3, 1e-45, 3.4028235e38, 0.1, 2.5, -7.0, 1e-8, 123456.789, 0.3])
    embs = {
        "small": np.float32([[0.5, 0.0], [0.5, 1.0], [0.5, 0.0]]),
        "tricky": tricky.reshape(3, 4),
        "random": rng.random((7, 5)).astype(np.float32) * np.float32(1e3),
        "empty_rows": np.zeros((0, 4), np.float32),
        "one_col": np.float32([[1 / 7], [2 / 7]]),
    }
    for name, z in embs.items():
        rec = {"name": name, "shape": list(z.shape), "z": b64(np.ascontiguousarray(z).tobytes())}
        for fmt in ("csv", "binary"):
            gee.write_embedding(z.astype(np.float64), path, fmt=fmt)
            rec[fmt] = b64(open(path, "rb").read())
        out["emb"].append(rec)
    base = base64.b64decode(out["emb"][2]["binary"])
    for name, data in [("bad_magic", b"XXXXXXXX" + base[8:]), ("truncated_header", base[:10]),
                       ("short_payload", base[:-8])]:
        with open(path, "wb") as fh:
            fh.write(data)
        out["emb"].append({"name": name, "data": b64(data), **outcome(lambda: gee.read_embedding(path).tolist(), path)})

    # write_edge_list / write_labels bytes
    for name, w in [("unit", None), ("weighted", np.float32([0.1, 2.5, 1e-7, 3e38, 1.0, 16777217.0]))]:
        src = np.int64([0, 5, 2, 9, 3, 1])
        dst = np.int64([1, 2, 7, 9, 0, 4])
        el = gee.EdgeList(n=10, src=src, dst=dst, w=np.ones(6) if w is None else w.astype(np.float64))
        gee.write_edge_list(el, path)
        out["write_edges"].append({"name": name, "src": src.tolist(), "dst": dst.tolist(),
                                   "w": None if w is None else b64(w.tobytes()), "text": b64(open(path, "rb").read())})
    y = gee.LabelVector(labels=np.int64([0, 3, 1, 0, 12]), k=12)
    gee.write_labels(y, path)
    out["write_labels"].append({"labels": [0, 3, 1, 0, 12], "text": b64(open(path, "rb").read())})

    # CLI generators: gen-er / gen-labels files (cli.py:134-146)
    from gee.cli import run_cli

    out["cli"] = []
    for argv in (["gen-er", "--nodes", "50", "--edges", "200", "--seed", "9"],
                 ["gen-er", "--nodes", "10", "--edges", "0", "--seed", "1"],
                 ["gen-labels", "--nodes", "40", "--k", "3", "--fraction", "0.5", "--seed", "2"]):
        assert run_cli(argv + ["--out", path]) == 0
        out["cli"].append({"argv": argv, "text": b64(open(path, "rb").read())})

    with open(os.path.join(HERE, "io_cases.json"), "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)
    print("wrote", os.path.join(HERE, "io_cases.json"))


if __name__ == "__main__":
    main()
