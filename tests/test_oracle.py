"""Pin the CPU oracle (oracle/) to the reference before trusting it.

Golden vectors come from running the reference itself
(tests/golden/make_golden.py); the known-answer tests restate the
reference's own (test_encoder.py, test_parallel.py, test_labeling.py).
CPU only.
"""

import numpy as np
import pytest

import oracle
from conftest import case, golden_cases

CHAIN_Z = [[0.5, 0.0], [0.5, 1.0], [0.5, 0.0]]


def test_golden_has_cases(golden):
    names = golden_cases(golden)
    assert {"chain", "mirror", "star", "two_hub", "self_loops", "empty", "unlabeled"} <= set(names)
    assert sum(n.startswith("rand") for n in names) == 10


def test_serial_oracle_bitwise_equals_reference(golden):
    # same arithmetic in the same order as serial_pass (_kernels.py:210-226)
    for name in golden_cases(golden):
        c = case(golden, name)
        z = oracle.serial_embed(c["src"], c["dst"], c["w"], c["labels"], int(c["n"]), int(c["k"]))
        assert np.array_equal(z, c["z_serial"]), name


def test_numpy_reference_matches_reference(golden):
    for name in golden_cases(golden):
        c = case(golden, name)
        z = oracle.numpy_reference(c["src"], c["dst"], c["w"], c["labels"], int(c["n"]), int(c["k"]))
        assert np.max(np.abs(z - c["z_serial"]), initial=0.0) <= 1e-9, name


def test_projection_matches_reference(golden):
    for name in golden_cases(golden):
        c = case(golden, name)
        counts, inv, row = oracle.projection(c["labels"], int(c["k"]))
        assert np.array_equal(counts[1:], c["class_counts"]), name
        assert np.array_equal(row, c["row_value"]), name


def test_projection_kats(golden):
    for i in range(6):
        c = case(golden, f"proj{i}")
        k = int(c["k"])
        counts, inv, row = oracle.projection(c["labels"], k)
        dense = np.zeros((c["labels"].size, k))
        idx = np.nonzero(c["labels"])[0]
        dense[idx, c["labels"][idx] - 1] = row[idx]
        assert np.array_equal(dense, c["dense"])
        assert np.array_equal(counts[1:], c["class_counts"])
    for i in range(5):
        c = case(golden, f"counts{i}")
        assert np.array_equal(oracle.bincount(c["labels"], int(c["k"])), c["bincount"])


def test_bincount_rejects_out_of_range():
    with pytest.raises(ValueError):
        oracle.bincount([0, 3], 2)


def test_build_csr_matches_reference(golden):
    for name in golden_cases(golden):
        c = case(golden, name)
        off, tgt, wts = oracle.build_csr(c["src"], c["dst"], c["w"], int(c["n"]), bool(c["directed"]))
        assert np.array_equal(off, c["csr_offsets"]), name
        assert np.array_equal(tgt, c["csr_targets"]), name
        assert np.array_equal(wts, c["csr_weights"]), name


@pytest.mark.parametrize("workers", [1, 2, 4, 8])
def test_parallel_port_matches_reference(golden, workers):
    for name in golden_cases(golden):
        c = case(golden, name)
        k = int(c["k"])
        w = None if np.all(c["csr_weights"] == 1.0) else c["csr_weights"]
        z = oracle.parallel_embed(c["csr_offsets"], c["csr_targets"], w, c["labels"], k, bool(c["directed"]), workers)
        assert np.max(np.abs(z - c["z_parallel"]), initial=0.0) <= 1e-9, (name, workers)
        assert np.max(np.abs(z - c["z_serial"]), initial=0.0) <= 1e-9, (name, workers)


def test_known_answers(golden):
    assert case(golden, "chain")["z_serial"].tolist() == CHAIN_Z
    assert case(golden, "mirror")["z_parallel"].tolist() == [[0.0, 1.0], [1.0, 0.0]]
    assert abs(case(golden, "star")["z_serial"][0, 0] - 1.0) <= 1e-12
    assert np.allclose(case(golden, "two_hub")["z_serial"][1:-1, 0], 1.0)
    assert not case(golden, "unlabeled")["z_serial"].any()
    assert not case(golden, "empty")["z_serial"].any()


def test_atomic_hammer_never_loses_updates():
    z = oracle.atomic_hammer(100000, 0.5, 8)  # test_parallel.py:67-79
    assert z[1] == 8 * 100000 * 0.5
    assert z[0] == 0.0


def test_sampled_rows_match_serial(golden):
    for name in golden_cases(golden):
        c = case(golden, name)
        n, k = int(c["n"]), int(c["k"])
        if not np.all(c["w"] == c["w"].astype(np.float32)):
            continue
        rows = np.arange(0, n, 3)
        zs = oracle.sampled_rows(c["src"], c["dst"], c["w"].astype(np.float32), c["labels"], k, rows)
        assert np.array_equal(zs, c["z_serial"][rows]), name


def test_race_graph_port_every_run(golden):
    c = case(golden, "two_hub")
    k = int(c["k"])
    for _ in range(20):
        z = oracle.parallel_embed(c["csr_offsets"], c["csr_targets"], None, c["labels"], k, True, 8)
        assert np.max(np.abs(z - c["z_serial"])) <= 1e-9


def test_random_labels_mirror_reproduces_reference_stream(golden):
    from paper_2402_04403_b200.labeling import random_labels

    for i in range(3):
        c = case(golden, f"rl{i}")
        n, k, seed = (int(x) for x in c["args"])
        assert np.array_equal(random_labels(n, k, float(c["fraction"]), seed).labels, c["labels"])


@pytest.mark.parametrize("scale,s,seed,first,weighted", [(10, 5000, 3, 0, True), (16, 20000, 77, 12345, False),
                                                         (27, 3000, 4, 10**9, True), (24, 4000, 3, 7, False)])
def test_c_rmat_generator_matches_numpy_restatement(scale, s, seed, first, weighted):
    # the reference arm builds C4 on the host with oracle.rmat_edges; it must
    # be the workload's own stream (synth.rmat_edges_numpy, itself pinned to
    # the GPU generator in tests/test_gpu_parity.py)
    from paper_2402_04403_b200 import synth

    got = oracle.rmat_edges(scale, s, seed, weighted=weighted, first=first, threads=3)
    exp = synth.rmat_edges_numpy(scale, s, seed, weighted=weighted, first=first)
    assert np.array_equal(got[0], exp[0]) and np.array_equal(got[1], exp[1])
    assert (got[2] is None) == (exp[2] is None)
    if weighted:
        assert np.array_equal(got[2], exp[2])
    assert np.array_equal(oracle.uniform_labels(7001, 50, seed), synth.uniform_labels_numpy(7001, 50, seed))


def test_parallel_directed_csr_is_the_reference_csr_up_to_row_order():
    rng = np.random.default_rng(9)
    n, s = 500, 20_000
    src, dst = rng.integers(0, n, s).astype(np.int32), rng.integers(0, n, s).astype(np.int32)
    w = rng.random(s).astype(np.float32)
    off, tgt, wt = oracle.build_csr_directed_par(src, dst, w, n, threads=4)
    ro, rt, rw = oracle.build_csr(src, dst, w, n, True)
    assert np.array_equal(off, ro)
    for r in range(n):
        a = sorted(zip(tgt[off[r]:off[r + 1]].tolist(), wt[off[r]:off[r + 1]].tolist()))
        b = sorted(zip(rt[ro[r]:ro[r + 1]].tolist(), rw[ro[r]:ro[r + 1]].tolist()))
        assert a == b
    y = rng.integers(0, 6, n)
    z1 = oracle.parallel_embed(off, tgt, wt, y, 5, True, 4)
    z2 = oracle.serial_embed(src, dst, w, y, n, 5)
    assert np.allclose(z1, z2, rtol=1e-12, atol=0)


def test_threaded_sampled_rows_and_mass_match_serial_oracle(rng):
    # the full-size config tests check sampled rows + column mass with this
    # threaded restatement; pin it to the serial oracle (signed weights,
    # unlabeled nodes, self loops, repeated edges)
    n, s, k = 4000, 50_000, 9
    src = rng.integers(0, n, s).astype(np.int32)
    dst = rng.integers(0, n, s).astype(np.int32)
    dst[:500] = src[:500]
    src[500:900] = 7
    w = rng.standard_normal(s).astype(np.float32)
    y = rng.integers(0, k + 1, n).astype(np.int32)
    z = oracle.serial_embed(src, dst, w, y, n, k)
    rows = np.unique(np.concatenate([rng.integers(0, n, 400), [7, 0, n - 1]]))
    for threads in (1, 6):
        zs, mass = oracle.sampled_rows_par(src, dst, w, y, k, rows, threads=threads)
        assert np.allclose(zs, z[rows], rtol=1e-12, atol=1e-12)
        assert np.allclose(mass, z.sum(0), rtol=1e-12, atol=1e-12)
    zs, mass = oracle.sampled_rows_par(src, dst, None, y, k, rows, threads=3)
    zu = oracle.serial_embed(src, dst, None, y, n, k)
    assert np.allclose(zs, zu[rows], rtol=1e-12, atol=0)
