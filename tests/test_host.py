"""Host-side logic and the C ABI surface (CPU only: no kernel launches)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_2402_04403_b200 as gb
from paper_2402_04403_b200 import _lib
from paper_2402_04403_b200.encoder import _check_out
from paper_2402_04403_b200.errors import ValidationError


def _declared_functions():
    names = []
    for h in ("gee_b200.h", "gee_synth.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names += re.findall(r"\b(gee_\w+)\s*\(", text)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared_functions()
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_pure_functions_without_gpu():
    L = _lib.lib
    assert L.gee_version() >= 100
    assert [L.gee_label_bytes(k) for k in (1, 255, 256, 65535, 65536)] == [1, 1, 2, 2, 4]
    assert L.gee_label_table_bytes(100, 0, 50) == 112 and L.gee_label_table_bytes(100, 20, 300) == 256
    # fixed-point exponent: |q| = max|w| 2^e < 2^41 (signed split planes) and
    # max row sum 2^e < 2^62
    e, rel = ctypes.c_int32(), ctypes.c_double()
    assert L.gee_block_scale_exp(1.0, 1.0, 2.0 ** -24, ctypes.byref(e), ctypes.byref(rel)) == 0
    assert e.value == 40 and rel.value == pytest.approx(2.0 ** -41 / 2.0 ** -24)
    assert L.gee_block_scale_exp(3.0, 0.999, 0.5, ctypes.byref(e), ctypes.byref(rel)) == 0
    assert 0.999 * 2.0 ** e.value < 2.0 ** 41 and 0.999 * 2.0 ** (e.value + 1) >= 2.0 ** 41
    assert L.gee_block_scale_exp(2.0 ** 30, 1.0, 0.5, ctypes.byref(e), ctypes.byref(rel)) == 0
    assert 2.0 ** 30 * 2.0 ** e.value < 2.0 ** 62 and e.value == 31
    # argument validation happens before any CUDA call
    assert L.gee_build_projection(None, 10, 0, None, None, None, None, None, 0, None, None) == _lib.GEE_ERR_INVALID
    assert b"positive" in L.gee_last_error()
    with pytest.raises(ValidationError):
        _lib.check(L.gee_embed_coo(None, None, None, 1, None, -1, None, 1, 5, None, 0, None))


def test_synth_word_matches_numpy_restatement():
    from paper_2402_04403_b200 import synth

    for seed, tag, ctr in [(0, 1, 0), (4, 2, 12345), (2**63 + 5, 4, 2**40)]:
        assert _lib.lib.gee_synth_word(seed, tag, ctr) == int(synth.word_numpy(seed, tag, np.uint64(ctr)))


def test_rmat_numpy_stream_shape():
    from paper_2402_04403_b200 import synth

    src, dst, w = synth.rmat_edges_numpy(10, 5000, seed=3, weighted=True)
    assert src.min() >= 0 and src.max() < 1024 and dst.max() < 1024
    assert w.min() > 0 and w.max() <= 1.0
    deg = np.bincount(src, minlength=1024)
    assert deg.max() > 20 * deg.mean()  # power-law hubs


def test_zipf_labels_sizes():
    from paper_2402_04403_b200 import synth

    y = synth.zipf_labels(4000, 10, 1.1, seed=5)
    counts = np.bincount(y, minlength=11)
    assert counts[0] == 0 and counts.sum() == 4000
    assert np.all(np.diff(counts[1:]) <= 0)


class TestContainers:
    def test_edge_list_validation(self):
        with pytest.raises(ValidationError):
            gb.EdgeList(n=2, src=[0], dst=[2])
        with pytest.raises(ValidationError):
            gb.EdgeList(n=2, src=[0, 1], dst=[1])
        with pytest.raises(ValidationError):
            gb.EdgeList(n=2, src=[0], dst=[1], w=[np.inf])
        with pytest.raises(ValidationError):
            gb.EdgeList(n=-1, src=[], dst=[])
        with pytest.raises(ValidationError):
            gb.EdgeList(n=2**31, src=[], dst=[])

    def test_edge_list_unit_weights(self):
        el = gb.EdgeList(n=3, src=[0, 1], dst=[1, 2], w=[1.0, 1.0])
        assert el.unit_weights and el.w is None and el.src.dtype == np.int32
        el = gb.EdgeList(n=3, src=[0, 1], dst=[1, 2], w=[1.0, 2.5])
        assert not el.unit_weights and el.w.dtype == np.float32

    def test_csr_validation(self):
        with pytest.raises(ValidationError):
            gb.CsrGraph(n=2, offsets=[0, 1], targets=[1])
        with pytest.raises(ValidationError):
            gb.CsrGraph(n=2, offsets=[0, 2, 1], targets=[1])
        with pytest.raises(ValidationError):
            gb.CsrGraph(n=2, offsets=[0, 1, 1], targets=[5])
        g = gb.CsrGraph(n=2, offsets=[0, 1, 1], targets=[1], weights=[1.0])
        assert g.unit_weights and g.s == 1

    def test_label_vector_validation(self):
        with pytest.raises(ValidationError, match="node 1"):
            gb.LabelVector(labels=[0, 5], k=2)
        with pytest.raises(ValidationError):
            gb.LabelVector(labels=[0, 1], k=0)

    def test_edge_accounting(self):
        g = gb.CsrGraph(n=2, offsets=[0, 1, 1], targets=[1], directed=True)
        assert gb.edge_accounting(g) is gb.EdgeAccounting.BOTH_ENDPOINTS
        assert gb.edge_accounting(g, directed=False) is gb.EdgeAccounting.SOURCE_ONLY

    def test_projection_matrix_dense(self):
        p = gb.ProjectionMatrix(3, 2, np.array([0.5, 0.5, 1.0]), np.array([1, 1, 2], dtype=np.int32))
        assert p.to_dense().tolist() == [[0.5, 0.0], [0.5, 0.0], [0.0, 1.0]]

    def test_out_validation(self):
        with pytest.raises(ValidationError):
            _check_out(np.zeros((2, 2)), 3, 2)
        with pytest.raises(ValidationError):
            _check_out(np.zeros((3, 2), dtype=np.int32), 3, 2)
        with pytest.raises(ValidationError):
            _check_out(np.zeros((2, 3)).T, 3, 2)
        assert _check_out(np.zeros((3, 2), dtype=np.float32), 3, 2) is not None

    def test_random_labels_contract(self):
        y = gb.random_labels(1003, 7, 0.25, seed=11)
        assert np.count_nonzero(y.labels) == round(0.25 * 1003)
        with pytest.raises(ValidationError):
            gb.random_labels(5, 3, 1.5, seed=1)


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2402_04403_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text, f


def test_weights_checked_before_float32_narrowing():
    # finite f64 weights float32 cannot carry are rejected with a specific
    # error instead of turning into inf / 0 (graph.py:46-47 checks finiteness
    # on the caller's f64 array)
    import paper_2402_04403_b200 as gb

    with pytest.raises(ValidationError, match="float32 range"):
        gb.EdgeList(n=2, src=[0], dst=[1], w=np.array([1e300]))
    with pytest.raises(ValidationError, match="normal float32 range"):
        gb.EdgeList(n=2, src=[0, 1], dst=[1, 0], w=np.array([1.0, 1e-300]))
    with pytest.raises(ValidationError, match="edge weights must be finite"):
        gb.EdgeList(n=2, src=[0], dst=[1], w=np.array([np.nan]))
    with pytest.raises(ValidationError, match="arc weights must be finite"):
        gb.CsrGraph(n=2, offsets=[0, 1, 1], targets=[1], weights=np.array([np.inf]))
    el = gb.EdgeList(n=2, src=[0, 1], dst=[1, 0], w=np.array([0.0, -2.5]))
    assert el.w.dtype == np.float32 and el.w.tolist() == [0.0, -2.5]


def test_bench_extra_steps_is_a_count_not_a_clock():
    """bench.py keeps the load up after the timed region for a number of
    steps derived from the (max-over-ranks) step time, never from a rank's
    own wall clock: the step holds collectives."""
    import importlib.util
    import os

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    assert bench.extra_steps(180.0, 10, 1) == 56  # 18 ms steps: about a second
    assert bench.extra_steps(1.0, 10, 1) == 2000  # capped
    assert bench.extra_steps(50000.0, 10, 1) == 1
    assert bench.extra_steps(0.0, 0, 1) == 2000
