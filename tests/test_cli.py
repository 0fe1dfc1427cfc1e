"""CLI contract (mirror of the reference's tests/test_cli.py and acceptance c10).

Usage / data errors and the generators run on CPU; embeds and the bench
subcommands need the GPU.  gen-er / gen-labels outputs are compared with the
files the reference's own CLI wrote for the same arguments
(tests/golden/io_cases.json, make_io_golden.py).
"""

import base64
import json
import os
import re

import numpy as np
import pytest

import paper_2402_04403_b200 as gb
from paper_2402_04403_b200.cli import run_cli

HERE = os.path.dirname(os.path.abspath(__file__))
CLI_GOLDEN = json.load(open(os.path.join(HERE, "golden", "io_cases.json")))["cli"]
CHAIN_Z = [[0.5, 0.0], [0.5, 1.0], [0.5, 0.0]]


def chain_files(tmp_path):
    graph = tmp_path / "chain.txt"
    graph.write_text("0 1\n1 2\n")
    labels = tmp_path / "chain.lab"
    labels.write_text("1\n1\n2\n")
    return graph, labels


# ------------------------------------------------------------------ CPU
def test_unknown_flag_is_usage_error(capsys):
    assert run_cli(["embed", "--frobnicate"]) == 1
    assert "error" in capsys.readouterr().err


def test_missing_required_option_is_usage_error(capsys):
    assert run_cli(["embed", "--graph", "g.txt"]) == 1
    capsys.readouterr()


def test_unknown_subcommand_is_usage_error(capsys):
    assert run_cli(["frobnicate"]) == 1
    capsys.readouterr()


def test_bad_device_is_usage_error(tmp_path, capsys):
    graph, labels = chain_files(tmp_path)
    assert run_cli(["embed", "--graph", str(graph), "--labels", str(labels), "--k", "2", "--device", "cpu",
                    "--out", str(tmp_path / "z.csv")]) == 1
    capsys.readouterr()


def test_missing_graph_is_data_error(tmp_path, capsys):
    code = run_cli(["embed", "--graph", str(tmp_path / "missing.txt"), "--labels", str(tmp_path / "missing.lab"),
                    "--k", "2", "--out", str(tmp_path / "z.csv")])
    assert code == 2
    assert "missing.txt" in capsys.readouterr().err


def test_bad_label_file_is_data_error(tmp_path, capsys):
    graph, _ = chain_files(tmp_path)
    labels = tmp_path / "bad.lab"
    labels.write_text("9\n9\n9\n")
    assert run_cli(["embed", "--graph", str(graph), "--labels", str(labels), "--k", "2",
                    "--out", str(tmp_path / "z.csv")]) == 2
    assert "outside [0, 2]" in capsys.readouterr().err


def test_parse_error_is_data_error(tmp_path, capsys):
    graph = tmp_path / "g.txt"
    graph.write_text("0 1\n1 x\n")
    _, labels = chain_files(tmp_path)
    assert run_cli(["embed", "--graph", str(graph), "--labels", str(labels), "--k", "2",
                    "--out", str(tmp_path / "z.csv")]) == 2
    assert "line 2: node ids must be integers" in capsys.readouterr().err


def test_embed_serial_rejects_cache(tmp_path, capsys):
    graph, labels = chain_files(tmp_path)
    cache = tmp_path / "chain.gee"
    el = gb.load_edge_list(graph)
    off = np.array([0, 1, 2, 2], np.int64)
    gb.write_binary_cache(gb.CsrGraph(n=3, offsets=off, targets=el.dst, directed=True), cache)
    code = run_cli(["embed", "--graph", str(cache), "--labels", str(labels), "--k", "2", "--serial",
                    "--out", str(tmp_path / "z.csv")])
    assert code == 2
    assert "text edge list" in capsys.readouterr().err


@pytest.mark.parametrize("case", CLI_GOLDEN, ids=[" ".join(c["argv"][:1] + c["argv"][2:4]) for c in CLI_GOLDEN])
def test_generators_match_reference_files(tmp_path, case, capsys):
    out = tmp_path / "f.txt"
    assert run_cli(case["argv"] + ["--out", str(out)]) == 0
    assert out.read_bytes() == base64.b64decode(case["text"])
    capsys.readouterr()


def test_gen_labels_counts(tmp_path, capsys):
    out = tmp_path / "y.txt"
    assert run_cli(["gen-labels", "--nodes", "40", "--k", "3", "--fraction", "0.5", "--seed", "2",
                    "--out", str(out)]) == 0
    values = [int(v) for v in out.read_text().split()]
    assert len(values) == 40 and sum(1 for v in values if v > 0) == 20
    assert "labeled=20" in capsys.readouterr().out


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_embed_serial_end_to_end(tmp_path, capsys):
    graph, labels = chain_files(tmp_path)
    out = tmp_path / "z.csv"
    assert run_cli(["embed", "--graph", str(graph), "--labels", str(labels), "--k", "2", "--serial",
                    "--out", str(out)]) == 0
    assert np.loadtxt(out, delimiter=",", ndmin=2).tolist() == CHAIN_Z
    summary = capsys.readouterr().out.strip().splitlines()[-1]
    assert re.fullmatch(r"n=3 s=2 k=2 workers=1 time_s=\d+\.\d{6}", summary)


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [[], ["--workers", "2"], ["--no-atomics"], ["--variant", "push"],
                                   ["--variant", "pull"], ["--gpus", "1"]])
def test_embed_parallel_matches_serial(tmp_path, extra, capsys):
    graph, labels = chain_files(tmp_path)
    out = tmp_path / "zp.csv"
    assert run_cli(["embed", "--graph", str(graph), "--labels", str(labels), "--k", "2", *extra,
                    "--out", str(out)]) == 0
    assert np.loadtxt(out, delimiter=",", ndmin=2).tolist() == CHAIN_Z
    capsys.readouterr()


@pytest.mark.gpu
def test_embed_binary_output_and_cache_input(tmp_path, capsys):
    graph, labels = chain_files(tmp_path)
    out = tmp_path / "z.bin"
    assert run_cli(["embed", "--graph", str(graph), "--labels", str(labels), "--k", "2", "--serial",
                    "--out", str(out), "--format", "binary"]) == 0
    assert gb.read_embedding(out).tolist() == CHAIN_Z
    for directed in (True, False):
        cache = tmp_path / f"chain{int(directed)}.gee"
        gb.write_binary_cache(gb.build_csr(gb.load_edge_list(graph, directed=directed)), cache)
        zc = tmp_path / "zc.csv"
        assert run_cli(["embed", "--graph", str(cache), "--labels", str(labels), "--k", "2", "--workers", "2",
                        "--out", str(zc)]) == 0
        assert np.loadtxt(zc, delimiter=",", ndmin=2).tolist() == CHAIN_Z
    capsys.readouterr()


@pytest.mark.gpu
def test_embed_weighted_text_matches_oracle(tmp_path, capsys):
    import oracle

    rng = np.random.default_rng(4)
    n, s, k = 3000, 40_000, 7
    src, dst = rng.integers(0, n, s), rng.integers(0, n, s)
    w = (1 - rng.random(s)).astype(np.float32)
    y = rng.integers(0, k + 1, n)
    graph, labels = tmp_path / "g.txt", tmp_path / "y.txt"
    gb.write_edge_list(gb.EdgeList(n=n, src=src, dst=dst, w=w), graph)
    gb.write_labels(gb.LabelVector(labels=y, k=k), labels)
    el = gb.load_edge_list(graph, weighted=True)
    expected = oracle.serial_embed(el.src, el.dst, el.w, y.astype(np.int32), el.n, k)
    for extra in ([], ["--serial"], ["--directed"]):
        out = tmp_path / "z.bin"
        assert run_cli(["embed", "--graph", str(graph), "--labels", str(labels), "--k", str(k), "--weighted",
                        *extra, "--out", str(out), "--format", "binary"]) == 0
        z = gb.read_embedding(out)
        nz = expected != 0
        assert np.all(z[~nz] == 0)
        assert np.max(np.abs(z[nz] - expected[nz]) / expected[nz]) <= 1e-4, extra
    capsys.readouterr()


@pytest.mark.gpu
@pytest.mark.parametrize("directed", [True, False])
@pytest.mark.parametrize("as_csr", [False, True])
def test_sharded_pass_is_bitwise_single_gpu(directed, as_csr):
    """Row shards (3 on one device here; one per GPU with --gpus N) write
    every Z row once: the result equals the single-GPU pull bit for bit."""
    import torch

    from paper_2402_04403_b200.multi import ShardedPass, embed_sharded

    rng = np.random.default_rng(12)
    n, s, k = 5000, 60_000, 9
    src = (rng.zipf(1.6, s) % n).astype(np.int32)  # skewed: hubs in the first shard
    dst = rng.integers(0, n, s).astype(np.int32)
    w = (1 - rng.random(s)).astype(np.float32)
    el = gb.EdgeList(n=n, src=src, dst=dst, w=w, directed=directed)
    y = gb.LabelVector(labels=rng.integers(0, k + 1, n), k=k)
    ref = gb.embed_serial(el, y, variant="pull")
    graph = gb.build_csr(el) if as_csr else el
    for shards in (1, 3):
        z = embed_sharded(graph, y, shards, devices=[0])
        assert np.array_equal(z, ref), shards
    sp = ShardedPass(graph, y, 2, devices=[0])
    ms = sp.run()
    assert list(ms) == [torch.device("cuda", 0)] and ms[torch.device("cuda", 0)] > 0
    assert np.array_equal(sp.gather(), ref)


@pytest.mark.gpu
def test_bench_scaling_writes_report(tmp_path, capsys):
    out = tmp_path / "report"
    assert run_cli(["bench-scaling", "--nodes", "2000", "--edges", "20000", "--seed", "3", "--k", "5",
                    "--gpus", "1", "--reps", "3", "--out", str(out)]) == 0
    lines = (out / "results.csv").read_text().splitlines()
    assert lines[0] == "name,n,s,k,workers,atomics,median_s,reps,gpus,variant,geps,roofline_frac"
    assert len(lines) == 2 and lines[1].startswith("er-20000,2000,20000,5,1,false,")
    assert "speedup(1)=1.00" in capsys.readouterr().out


@pytest.mark.gpu
def test_bench_sweep_writes_report(tmp_path, capsys):
    out = tmp_path / "report"
    assert run_cli(["bench-sweep", "--sizes", "20000,40000", "--n-per-s", "0.05", "--k", "5", "--seed", "3",
                    "--reps", "3", "--out", str(out)]) == 0
    assert len((out / "results.csv").read_text().splitlines()) == 3
    assert "linear fit" in capsys.readouterr().out


@pytest.mark.gpu
@pytest.mark.parametrize("as_csr", [False, True])
def test_sharded_pass_wide_weight_range_falls_back_to_push(tmp_path, as_csr):
    """Weights whose merged range fails the exact pull's fixed-point gate:
    the row shards push their own rows (SOURCE_ONLY) instead of raising;
    Z matches the f64 oracle within the push tolerance, and the CLI's
    `embed --gpus 2` runs on such a graph."""
    import oracle

    from paper_2402_04403_b200.multi import ShardedPass

    rng = np.random.default_rng(33)
    n, s, k = 4000, 50_000, 7
    src = (rng.zipf(1.6, s) % n).astype(np.int32)
    dst = rng.integers(0, n, s).astype(np.int32)
    w = (1 - rng.random(s)).astype(np.float32)
    w[::97] = 1e-12  # one shard alone may pass the gate; the whole graph does not
    el = gb.EdgeList(n=n, src=src, dst=dst, w=w, directed=True)
    y = gb.LabelVector(labels=rng.integers(0, k + 1, n), k=k)
    exp = oracle.serial_embed(src, dst, w, y.labels, n, k)
    graph = gb.build_csr(el) if as_csr else el
    sp = ShardedPass(graph, y, 2, devices=[0])
    assert sp.variant == "push"
    sp.run()
    z = sp.gather()
    nz = exp != 0
    assert np.all(z[~nz] == 0)
    assert np.max(np.abs(z[nz] - exp[nz]) / np.abs(exp[nz])) <= 1e-4
    import torch

    if torch.cuda.device_count() >= 2:  # the CLI places one shard per visible GPU
        edges, labels, out = tmp_path / "wide.txt", tmp_path / "y.txt", tmp_path / "z.bin"
        gb.write_edge_list(el, edges)
        gb.write_labels(y, labels)
        assert run_cli(["embed", "--graph", str(edges), "--labels", str(labels), "--k", str(k), "--weighted",
                        "--directed", "--gpus", "2", "--out", str(out), "--format", "binary"]) == 0


@pytest.mark.gpu
def test_sharded_histogram_kernel_sums_to_full_projection():
    """gee_build_projection_sharded: per-rank label slices' counts sum to
    the full histogram and every rank's label table equals the replicated
    one (bench.py's row-range run)."""
    import torch

    from paper_2402_04403_b200 import synth
    from paper_2402_04403_b200.device import DeviceGraph, Embedder
    from paper_2402_04403_b200.shard import label_slice

    scale, s, k = 15, 300_000, 50
    n = 1 << scale
    src, dst, w = synth.rmat_edges(scale, s, seed=2, weighted=True, device="cuda")
    y = synth.uniform_labels(n, k, seed=2, device="cuda")
    y[::11] = 0
    g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
    g.prepare_hot(k, enable=True)
    full = Embedder(n, k)
    full.project(y, g=g)
    ref_counts, ref_table, ref_inv = full.counts.clone(), full.table.clone(), full.inv64.clone()
    for world in (2, 3):
        tot = torch.zeros_like(ref_counts)
        for rank in range(world):
            emb = Embedder(n, k)
            lo, hi = label_slice(n, world, rank)
            parts = []
            emb.project_sharded(y, g, lo, hi, lambda c: parts.append(c.clone()))
            tot += parts[0]
            used = g.n_hot + n + 1  # the rest is alignment padding
            assert torch.equal(emb.table[:used], ref_table[:used])
        assert torch.equal(tot, ref_counts)
    emb = Embedder(n, k)
    emb.project_sharded(y, g, 0, n, lambda c: c)
    assert torch.equal(emb.counts, ref_counts) and torch.equal(emb.inv64, ref_inv)
    z = emb.pull(g)
    assert torch.equal(z, full.pull(g))
