"""Data formats through libgee_io.so against the reference's own outcomes.

tests/golden/io_cases.json was produced by running the reference's readers
and writers on every input below (tests/golden/make_io_golden.py): parsed
arrays, written bytes, or exception type + text.  Host-only (no GPU).
"""

import base64
import json
import os

import numpy as np
import pytest

import paper_2402_04403_b200 as gb
from paper_2402_04403_b200 import formats
from paper_2402_04403_b200.errors import FormatError, ParseError, ValidationError

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "io_cases.json")))
ERRORS = {"ParseError": ParseError, "FormatError": FormatError, "ValidationError": ValidationError}


def _b(s):
    return base64.b64decode(s)


def _write(tmp_path, data, name="f"):
    p = tmp_path / name
    p.write_bytes(data)
    return p


def _expect_error(case, path, fn):
    with pytest.raises(ERRORS[case["error"]]) as ei:
        fn()
    assert str(ei.value) == case["message"].replace("{path}", str(path))


@pytest.mark.parametrize("case", CASES["edges"], ids=[c["name"] for c in CASES["edges"]])
@pytest.mark.parametrize("threads", [1, 8])
def test_load_edge_list_matches_reference(tmp_path, case, threads):
    p = _write(tmp_path, _b(case["data"]))
    if "error" in case:
        _expect_error(case, p, lambda: gb.load_edge_list(p, weighted=case["weighted"], threads=threads))
        _expect_error(case, p, lambda: formats.load_edge_list_f64(p, weighted=case["weighted"], threads=threads))
        return
    ref = case["ok"]
    el = gb.load_edge_list(p, weighted=case["weighted"], directed=False, threads=threads)
    assert el.n == ref["n"] and el.directed is False
    assert el.src.tolist() == ref["src"] and el.dst.tolist() == ref["dst"]
    assert el.weights().tolist() == np.float32(ref["w"]).tolist()  # fp32 of the reference's f64
    n, src, dst, w = formats.load_edge_list_f64(p, weighted=case["weighted"], threads=threads)
    assert n == ref["n"] and src.tolist() == ref["src"] and dst.tolist() == ref["dst"]
    assert w.tolist() == ref["w"]  # bit-exact f64 parse (Python float() == strtod, correctly rounded)


@pytest.mark.parametrize("case", CASES["labels"], ids=[c["name"] for c in CASES["labels"]])
def test_load_labels_matches_reference(tmp_path, case):
    p = _write(tmp_path, _b(case["data"]))
    if "error" in case:
        _expect_error(case, p, lambda: gb.load_labels(p, case["n"], case["k"]))
        return
    y = gb.load_labels(p, case["n"], case["k"])
    assert y.labels.tolist() == case["ok"] and y.k == case["k"]


@pytest.mark.parametrize("case", CASES["csr"], ids=[c["name"] for c in CASES["csr"]])
def test_binary_cache_matches_reference(tmp_path, case):
    p = _write(tmp_path, _b(case["data"]), "g.bin")
    if "error" in case:
        _expect_error(case, p, lambda: gb.read_binary_cache(p))
        return
    g = gb.read_binary_cache(p, threads=4)
    assert g.n == case["n"] and g.directed == case["directed"]
    assert g.offsets.tolist() == case["offsets"] and g.targets.tolist() == case["targets"]
    w = np.ones(g.s, np.float32) if g.weights is None else g.weights
    assert w.tolist() == np.float32(case["weights"]).tolist()
    # writing it back gives the reference's bytes
    q = tmp_path / "back.bin"
    gb.write_binary_cache(g, q)
    assert q.read_bytes() == _b(case["data"])


@pytest.mark.parametrize("case", CASES["emb"], ids=[c["name"] for c in CASES["emb"]])
def test_embedding_formats_match_reference(tmp_path, case):
    if "error" in case:
        p = _write(tmp_path, _b(case["data"]), "z.bin")
        _expect_error(case, p, lambda: gb.read_embedding(p))
        return
    z = np.frombuffer(_b(case["z"]), np.float32).reshape(case["shape"])
    for fmt in ("csv", "binary"):
        p = tmp_path / f"z.{fmt}"
        gb.write_embedding(z, p, fmt=fmt, threads=3)
        assert p.read_bytes() == _b(case[fmt]), fmt
        gb.write_embedding(z.astype(np.float64), p, fmt=fmt)
        assert p.read_bytes() == _b(case[fmt]), fmt + " (f64 input)"
    back = gb.read_embedding(tmp_path / "z.binary")
    assert back.dtype == np.float64 and np.array_equal(back, z.astype(np.float64))


def test_embedding_errors(tmp_path):
    with pytest.raises(ValidationError, match="2-d"):
        gb.write_embedding(np.zeros(3), tmp_path / "x")
    with pytest.raises(ValidationError) as ei:
        gb.write_embedding(np.zeros((2, 2)), tmp_path / "x", fmt="parquet")
    assert str(ei.value) == "unknown embedding format 'parquet'"
    with pytest.raises(FileNotFoundError):
        gb.read_embedding(tmp_path / "missing.bin")


@pytest.mark.parametrize("case", CASES["write_edges"], ids=[c["name"] for c in CASES["write_edges"]])
def test_write_edge_list_matches_reference(tmp_path, case):
    w = None if case["w"] is None else np.frombuffer(_b(case["w"]), np.float32)
    el = gb.EdgeList(n=10, src=np.int32(case["src"]), dst=np.int32(case["dst"]), w=w)
    p = tmp_path / "e.txt"
    gb.write_edge_list(el, p)
    assert p.read_bytes() == _b(case["text"])
    back = gb.load_edge_list(p, weighted=w is not None)
    assert back.src.tolist() == case["src"] and back.dst.tolist() == case["dst"]
    if w is not None:
        assert np.array_equal(back.w, w)  # repr round-trips exactly


def test_write_labels_matches_reference(tmp_path):
    case = CASES["write_labels"][0]
    p = tmp_path / "y.txt"
    gb.write_labels(gb.LabelVector(labels=np.int32(case["labels"]), k=12), p)
    assert p.read_bytes() == _b(case["text"])


def test_missing_file_is_oserror(tmp_path):
    with pytest.raises(FileNotFoundError) as ei:
        gb.load_edge_list(tmp_path / "nope.txt")
    assert "No such file or directory" in str(ei.value)
    with pytest.raises(IsADirectoryError):
        gb.load_labels(tmp_path, 3, 2)


def _big_edge_text(rng, s, n, weighted):
    src = rng.integers(0, n, s)
    dst = rng.integers(0, n, s)
    w = rng.random(s).astype(np.float32) if weighted else None
    el = gb.EdgeList(n=n, src=src, dst=dst, w=w)
    return el, src, dst, w


def test_multichunk_parse_and_error_line(tmp_path):
    """A file large enough for many worker chunks: same arrays as the
    generator, and the reported error line is the first bad line in file
    order even when later chunks also hold errors."""
    rng = np.random.default_rng(3)
    s, n = 600_000, 1 << 20
    el, src, dst, w = _big_edge_text(rng, s, n, True)
    p = tmp_path / "big.txt"
    gb.write_edge_list(el, p)
    for threads in (1, 16):
        got = gb.load_edge_list(p, weighted=True, threads=threads)
        assert np.array_equal(got.src, src.astype(np.int32)) and np.array_equal(got.dst, dst.astype(np.int32))
        assert np.array_equal(got.w, w)
        assert got.n == int(max(src.max(), dst.max())) + 1
    lines = p.read_bytes().split(b"\n")
    lines[400_123] = b"1 2 nope"
    lines[500_000] = b"-5 2 1.0"
    lines[123] = b"# comment moves nothing"
    bad = tmp_path / "bad.txt"
    bad.write_bytes(b"\n".join(lines))
    for threads in (1, 16):
        with pytest.raises(ParseError) as ei:
            gb.load_edge_list(bad, weighted=True, threads=threads)
        assert str(ei.value) == f"{bad}: line 400124: weight is not a number"
    # \r\n line ends across chunk boundaries keep the numbering
    crlf = tmp_path / "crlf.txt"
    crlf.write_bytes(b"\r\n".join(lines))
    with pytest.raises(ParseError) as ei:
        gb.load_edge_list(crlf, weighted=True, threads=16)
    assert str(ei.value) == f"{crlf}: line 400124: weight is not a number"


def test_multichunk_labels(tmp_path):
    rng = np.random.default_rng(5)
    n, k = 700_000, 50
    lab = rng.integers(0, k + 1, n).astype(np.int32)
    p = tmp_path / "y.txt"
    gb.write_labels(gb.LabelVector(labels=lab, k=k), p)
    y = gb.load_labels(p, n, k, threads=16)
    assert np.array_equal(y.labels, lab)
    lines = p.read_bytes().split(b"\n")
    lines[654_321] = b"3 4"
    q = tmp_path / "mixed.txt"
    q.write_bytes(b"\n".join(lines))
    with pytest.raises(ParseError) as ei:
        gb.load_labels(q, n, k, threads=16)
    assert str(ei.value) == f"{q}: line 654322: mixed label formats"


def test_binary_cache_round_trip_large(tmp_path):
    rng = np.random.default_rng(11)
    n, s = 100_000, 2_000_000
    deg = np.bincount(rng.integers(0, n, s), minlength=n)
    offsets = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    targets = rng.integers(0, n, s).astype(np.int32)
    w = rng.random(s).astype(np.float32)
    g = gb.CsrGraph(n=n, offsets=offsets, targets=targets, weights=w, directed=False)
    p = tmp_path / "g.bin"
    gb.write_binary_cache(g, p, threads=8)
    assert p.stat().st_size == 26 + 8 * (n + 1) + 12 * s
    back = gb.read_binary_cache(p, threads=8)
    assert not back.directed and np.array_equal(back.offsets, offsets)
    assert np.array_equal(back.targets, targets) and np.array_equal(back.weights, w)


def test_io_library_exports_every_header_symbol():
    import re

    hdr = open(os.path.join(os.path.dirname(HERE), "include", "gee_io.h")).read()
    declared = set(re.findall(r"\b(gee_io_\w+)\s*\(", hdr))
    assert declared == set(formats.IO_SIGNATURES), declared ^ set(formats.IO_SIGNATURES)
    lib = formats.io_lib()
    for name in declared:
        assert hasattr(lib, name)


def test_weight_repr_matches_python(tmp_path):
    """write_edge_list formats weights as repr(float(w)) (graph.py:155):
    random fp32 bit patterns across every exponent, plus the edges."""
    rng = np.random.default_rng(9)
    bits = rng.integers(0, 2**32, 50_000, dtype=np.uint64).astype(np.uint32)
    w = bits.view(np.float32)
    w = w[np.isfinite(w)]
    w = np.concatenate([w, np.float32([0.0, -0.0, 1.0, 1e16, 1e-5, 1e-4, 9.999999e15, 1e15, 0.1, 2.0**-149])])
    s = w.shape[0]
    el = gb.EdgeList(n=2, src=np.zeros(s, np.int32), dst=np.ones(s, np.int32), w=w)
    p = tmp_path / "w.txt"
    gb.write_edge_list(el, p, threads=4)
    got = [ln.split(" ")[2] for ln in p.read_text().splitlines()]
    assert got == [repr(float(x)) for x in w]


@pytest.mark.parametrize("scalar", [False, True])
@pytest.mark.parametrize("rows,k", [(1, 1), (3000, 50), (2048, 64), (1500, 130), (700, 17), (1100, 200), (0, 5)])
def test_expand_rows_rebuilds_dense_z(rows, k, scalar, monkeypatch):
    """gee_io_expand_rows (the host half of the streamed pass's row-sparse
    Z copy) from the format built in numpy: u64 row masks, packed nonzeros,
    per-1024-row value offsets; every bit pattern survives, -0.0 included.
    Both the AVX-512 expand-load path (where the CPU has it) and the scalar
    path (GEE_IO_SCALAR=1)."""
    monkeypatch.setenv("GEE_IO_SCALAR", "1" if scalar else "0")
    rng = np.random.default_rng(rows * 7 + k)
    z = np.where(rng.random((rows, k)) < 0.2, rng.standard_normal((rows, k)), 0.0).astype(np.float32)
    if rows:
        z[0, -1] = -0.0
    nz = z.view(np.uint32) != 0
    mw = (k + 63) // 64
    bits = np.zeros((rows, mw * 64), bool)
    bits[:, :k] = nz
    mask = np.packbits(bits.reshape(rows, mw, 64)[..., ::-1], axis=-1).view(">u8").reshape(rows, mw).astype(np.uint64)
    vals = z[nz].copy()
    nb = (rows + 1023) // 1024
    boff = np.concatenate([[0], np.cumsum(nz.sum(1))])[::1024][:nb].astype(np.int64)
    boff = np.concatenate([boff, [nz.sum()]]).astype(np.int64)
    out = np.full((rows, k), np.nan, np.float32)
    lib = formats.io_lib()
    assert lib.gee_io_expand_rows(mask.ctypes.data, vals.ctypes.data, boff.ctypes.data, rows, k, out.ctypes.data,
                                  4) == 0
    assert np.array_equal(out.view(np.uint32), z.view(np.uint32))
