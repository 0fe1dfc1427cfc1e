"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle.

Bar (BASELINE.json north_star):
  * class counts bit-exact;
  * Z max relative error <= 1e-4 per entry vs the f64 oracle, entries that
    are zero in the oracle exactly zero;
  * exact equality where the values are fp32-representable (chain, mirror,
    two-hub, hammer);
  * the pull variant bit-stable run to run.
"""

import ctypes
import numpy as np
import pytest

import oracle
from conftest import case, golden_cases, rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2402_04403_b200 as gb  # noqa: E402
from paper_2402_04403_b200 import synth  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph, Embedder  # noqa: E402

TOL = 1e-4  # max relative error vs the f64 oracle (fp32 Z)

EXACT_CASES = ("chain", "mirror", "two_hub", "star_exact", "self_loops", "empty", "unlabeled")


def _el(c):
    w = c["w"]
    return gb.EdgeList(n=int(c["n"]), src=c["src"], dst=c["dst"], w=w, directed=bool(c["directed"]))


def _y(c):
    return gb.LabelVector(labels=c["labels"], k=int(c["k"]))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("variant", ["pull", "push"])
def test_golden_embed_serial(golden, variant):
    for name in golden_cases(golden):
        c = case(golden, name)
        z = gb.embed_serial(_el(c), _y(c), variant=variant)
        assert z.dtype == np.float32 and z.shape == c["z_serial"].shape
        assert rel_err(z, c["z_serial"]) <= TOL, (name, variant)
        if name in ("chain", "mirror", "two_hub", "self_loops", "empty", "unlabeled"):
            assert np.array_equal(z.astype(np.float64), c["z_serial"]), (name, variant)


@pytest.mark.parametrize("variant", ["pull", "push"])
def test_golden_embed_parallel_on_reference_csr(golden, variant):
    for name in golden_cases(golden):
        c = case(golden, name)
        g = gb.CsrGraph(n=int(c["n"]), offsets=c["csr_offsets"], targets=c["csr_targets"],
                        weights=c["csr_weights"], directed=bool(c["directed"]))
        z = gb.embed_parallel(g, _y(c), workers=8, variant=variant)
        assert rel_err(z, c["z_parallel"]) <= TOL, (name, variant)
        assert rel_err(z, c["z_serial"]) <= TOL, (name, variant)


def test_class_counts_bit_exact(golden):
    for name in golden_cases(golden):
        c = case(golden, name)
        assert np.array_equal(gb.class_counts(_y(c)), c["class_counts"]), name
    for i in range(5):
        c = case(golden, f"counts{i}")
        y = gb.LabelVector(labels=c["labels"], k=int(c["k"]))
        assert np.array_equal(gb.class_counts(y), c["bincount"][1:])


def test_projection_kats(golden):
    for i in range(6):
        c = case(golden, f"proj{i}")
        p = gb.build_projection(gb.LabelVector(labels=c["labels"], k=int(c["k"])))
        assert np.array_equal(p.to_dense(), c["dense"])


def test_projection_warnings(caplog):
    with caplog.at_level("WARNING", logger="paper_2402_04403_b200.encoder"):
        gb.build_projection(gb.LabelVector(labels=[1, 1], k=3))
    assert "no members" in caplog.text
    with caplog.at_level("WARNING", logger="paper_2402_04403_b200.encoder"):
        gb.build_projection(gb.LabelVector(labels=[0, 0], k=2))
    assert "identically zero" in caplog.text


def test_build_csr_matches_reference_order(golden):
    for name in golden_cases(golden):
        c = case(golden, name)
        g = gb.build_csr(_el(c), stable=True)
        assert np.array_equal(g.offsets, c["csr_offsets"]), name
        assert np.array_equal(g.targets, c["csr_targets"]), name
        w = np.ones(g.s) if g.weights is None else g.weights
        assert np.array_equal(np.asarray(w, dtype=np.float64), c["csr_weights"]), name


def test_pull_bit_stable(golden):
    for name in ("rand1", "rand2", "rand4", "rand5"):
        c = case(golden, name)
        a = gb.embed_serial(_el(c), _y(c), variant="pull")
        b = gb.embed_serial(_el(c), _y(c), variant="pull")
        assert np.array_equal(a, b), name


def test_star_closed_form():
    leaves = 1000
    el = gb.EdgeList(n=leaves + 1, src=np.zeros(leaves), dst=np.arange(1, leaves + 1), directed=False)
    y = gb.LabelVector(labels=[0] + [1] * leaves, k=1)
    g = gb.build_csr(el)
    for variant in ("pull", "push"):
        z = gb.embed_parallel(g, y, variant=variant)
        assert abs(z[0, 0] - 1.0) <= TOL  # fp32: 1000 * fl(1/1000) != 1 exactly (push)
        assert not z[1:].any()


def two_hub(leaves):
    n = leaves + 2
    ids = np.arange(1, leaves + 1)
    src = np.concatenate([np.zeros(leaves, np.int64), np.full(leaves, n - 1)])
    dst = np.concatenate([ids, ids])
    labels = np.zeros(n, dtype=np.int64)
    labels[0] = labels[n - 1] = 1
    return gb.EdgeList(n=n, src=src, dst=dst, directed=True), gb.LabelVector(labels=labels, k=2)


@pytest.mark.parametrize("variant", ["pull", "push"])
def test_race_graph_every_run(variant):
    el, y = two_hub(100_000)
    expected = oracle.serial_embed(el.src, el.dst, None, y.labels, el.n, y.k)
    assert np.allclose(expected[1:-1, 0], 1.0)
    dev = torch.device("cuda")
    g = DeviceGraph.from_edges(el.src, el.dst, None, el.n, device=dev, pull=variant == "pull",
                               keep_coo=variant == "push")
    emb = Embedder(el.n, y.k, dev)
    lab = torch.from_numpy(y.labels).to(dev)
    z = emb.new_z()
    for _ in range(100):
        emb.embed(g, lab, variant=variant, z=z)
        assert np.array_equal(z.cpu().numpy().astype(np.float64), expected)


def test_red_hammer_exact():
    # every edge hits Z[0, 0]; 0.5 increments stay exact in fp32
    s = 800_000
    el = gb.EdgeList(n=2, src=np.zeros(s), dst=np.ones(s), w=np.full(s, 0.5), directed=True)
    y = gb.LabelVector(labels=[0, 1], k=1)
    for variant in ("push", "pull"):
        z = gb.embed_serial(el, y, variant=variant)
        assert z[0, 0] == s * 0.5 and z[1, 0] == 0.0, variant


def test_out_buffer_reused_and_validated(golden):
    c = case(golden, "chain")
    g = gb.CsrGraph(n=3, offsets=c["csr_offsets"], targets=c["csr_targets"], weights=c["csr_weights"])
    out = np.full((3, 2), 7.0)
    z = gb.embed_parallel(g, _y(c), workers=2, out=out)
    assert z is out and out.tolist() == c["z_serial"].tolist()
    out_d = torch.full((3, 2), 7.0, device="cuda")
    z = gb.embed_parallel(g, _y(c), out=out_d)
    assert z is out_d and z.cpu().numpy().tolist() == c["z_serial"].tolist()
    with pytest.raises(gb.ValidationError):
        gb.embed_parallel(g, _y(c), out=np.zeros((2, 2)))
    with pytest.raises(gb.ValidationError):
        gb.embed_parallel(g, _y(c), workers=0)
    with pytest.raises(gb.ValidationError):
        gb.embed_parallel(g, gb.LabelVector(labels=[1], k=2))
    with pytest.raises(gb.ValidationError):
        gb.embed_serial(_el(c), gb.LabelVector(labels=[1, 2], k=2))


def test_device_tensors_in_device_tensor_out(golden):
    c = case(golden, "rand4")
    dev = torch.device("cuda")
    z = gb.embed(torch.from_numpy(c["src"]).to(dev), torch.from_numpy(c["dst"]).to(dev),
                 torch.from_numpy(c["labels"]).to(dev), int(c["n"]), int(c["k"]),
                 weights=torch.from_numpy(c["w"]).to(dev), directed=bool(c["directed"]))
    assert isinstance(z, torch.Tensor) and z.is_cuda
    assert rel_err(z.cpu().numpy(), c["z_serial"]) <= TOL


def test_synth_gpu_matches_numpy_restatement():
    s, scale, seed = 20000, 16, 77
    src, dst, w = synth.rmat_edges(scale, s, seed, weighted=True, first=12345)
    es, ed, ew = synth.rmat_edges_numpy(scale, s, seed, weighted=True, first=12345)
    assert np.array_equal(src.cpu().numpy(), es) and np.array_equal(dst.cpu().numpy(), ed)
    assert np.array_equal(w.cpu().numpy(), ew)
    src, dst, w = synth.er_edges(1000003, s, seed, weighted=True)
    es, ed, ew = synth.er_edges_numpy(1000003, s, seed, weighted=True)
    assert np.array_equal(src.cpu().numpy(), es) and np.array_equal(dst.cpu().numpy(), ed)
    assert np.array_equal(w.cpu().numpy(), ew)
    y = synth.uniform_labels(5000, 50, seed)
    assert np.array_equal(y.cpu().numpy(), synth.uniform_labels_numpy(5000, 50, seed))


def test_empty_and_trailing_rows():
    # rows after the last arc and isolated rows in between must be zero
    el = gb.EdgeList(n=10, src=[2, 3], dst=[3, 2], w=[1.0, 2.0])
    y = gb.LabelVector(labels=[1] * 10, k=1)
    for variant in ("pull", "push"):
        z = gb.embed_serial(el, y, variant=variant)
        exp = oracle.serial_embed(el.src, el.dst, el.w, y.labels, 10, 1)
        assert rel_err(z, exp) <= TOL


def _check_random(rng, n, s, k, weighted, directed, frac, variant):
    src = rng.integers(0, n, s)
    dst = rng.integers(0, n, s)
    w = (2.0 * (1.0 - rng.random(s))).astype(np.float32) if weighted else None
    y = gb.random_labels(n, k, frac, int(rng.integers(0, 2**31)))
    el = gb.EdgeList(n=n, src=src, dst=dst, w=w, directed=directed)
    z = gb.embed_serial(el, y, variant=variant)
    exp = oracle.serial_embed(src, dst, w, y.labels, n, k)
    assert rel_err(z, exp) <= TOL


@pytest.mark.parametrize("variant", ["pull", "push"])
def test_random_battery(variant):
    # test_acceptance.py:77-98 shapes, restated to the fp32 tolerance
    rng = np.random.default_rng(2024)
    for i in range(30):
        n = int(rng.integers(2, 10_001))
        s = int(rng.integers(0, 100_001))
        _check_random(rng, n, s, (2, 10, 50, 300, 1000)[i % 5], bool(i % 3), bool(i % 2), (0.1, 1.0)[i % 2], variant)


def test_hub_rows_span_many_tiles():
    # one row with 100k arcs crosses ~25 pull tiles; plus a dense cluster
    rng = np.random.default_rng(7)
    n, k = 5000, 20
    src = np.concatenate([np.zeros(100_000, np.int64), rng.integers(0, n, 50_000)])
    dst = np.concatenate([rng.integers(0, n, 100_000), rng.integers(0, 50, 50_000)])
    w = (1.0 - rng.random(src.size)).astype(np.float32)
    y = gb.random_labels(n, k, 0.7, 5)
    el = gb.EdgeList(n=n, src=src, dst=dst, w=w, directed=True)
    exp = oracle.serial_embed(src, dst, w, y.labels, n, k)
    for variant in ("pull", "push"):
        assert rel_err(gb.embed_serial(el, y, variant=variant), exp) <= TOL, variant


def test_mass_accounting():
    rng = np.random.default_rng(5)
    for i in range(10):
        n = int(rng.integers(2, 3000))
        s = int(rng.integers(1, 30_000))
        src, dst = rng.integers(0, n, s), rng.integers(0, n, s)
        w = (2.0 * (1.0 - rng.random(s))).astype(np.float32)
        y = gb.random_labels(n, 10, 0.1, seed=i)
        _, inv, row = oracle.projection(y.labels, 10)
        lab = y.labels
        mass = np.where(lab[dst] > 0, row[dst] * w, 0.0).sum() + np.where(lab[src] > 0, row[src] * w, 0.0).sum()
        z = gb.embed_serial(gb.EdgeList(n=n, src=src, dst=dst, w=w, directed=bool(i % 2)), y)
        assert abs(z.astype(np.float64).sum() - mass) <= 1e-5 * max(1.0, abs(mass))


@pytest.mark.parametrize("k,weighted", [(50, True), (300, False), (5, False)])
def test_hot_tier_all_three_label_paths(k, weighted):
    # forced hot tier on a skewed graph: shared-memory head, L2 table and
    # cold packed labels are all exercised (n_hot exceeds the smem head)
    scale, s = 19, 4_000_000
    src, dst, w = synth.rmat_edges(scale, s, seed=11, weighted=weighted)
    n = 1 << scale
    y = synth.uniform_labels(n, k, seed=12)
    dev = torch.device("cuda")
    g = DeviceGraph.from_edges(src, dst, w, n, device=dev, pull=True)
    g.prepare_hot(k, enable=True)
    assert g.n_hot > 120_000 and g.n_hot < n
    emb = Embedder(n, k, dev)
    z = emb.embed(g, y, variant="pull").cpu().numpy()
    exp = oracle.serial_embed(src.cpu().numpy(), dst.cpu().numpy(), None if w is None else w.cpu().numpy(),
                              y.cpu().numpy(), n, k)
    assert rel_err(z, exp) <= TOL
    z2 = emb.embed(g, y, variant="pull").cpu().numpy()
    assert np.array_equal(z, z2)  # bit-stable


def test_hot_plan_ranks_by_degree():
    src = np.array([0, 0, 0, 1, 1, 2, 5, 5, 5, 5], dtype=np.int64)
    dst = np.array([1, 2, 3, 2, 3, 3, 4, 4, 4, 4], dtype=np.int64)
    dev = torch.device("cuda")
    g = DeviceGraph.from_edges(src, dst, None, 6, device=dev, pull=True)
    g.prepare_hot(3, enable=True)
    deg = np.bincount(np.concatenate([src, dst]), minlength=6)
    rank = g.hot_rank.cpu().numpy()
    order = sorted(range(6), key=lambda v: (-deg[v], v))
    hot = [v for v in order if deg[v] >= 2]
    assert g.n_hot == len(hot)
    for r, v in enumerate(hot):
        assert rank[v] == r
    assert all(rank[v] == -1 for v in range(6) if deg[v] < 2)


def _force_wide(monkeypatch):
    monkeypatch.setattr(Embedder, "reducer_for", lambda self, g, z=None: "wide")


@pytest.mark.parametrize("k,weighted", [(50, True), (7, False), (2, True), (255, False)])
def test_pull_reducers_agree_bitwise(k, weighted, monkeypatch):
    # both exact pull paths (class stream + 32-row block reducer + heavy
    # items; the fused wide kernel) sum the same integers: their Z must match
    # bit for bit.  The graph mixes empty rows, dense blocks (several window
    # passes), a heavy row inside a block and ragged tails.
    rng = np.random.default_rng(k)
    n = 40_003
    hub = np.full(30_000, 37, np.int64)
    src = np.concatenate([hub, rng.integers(0, n // 3, 200_000), np.arange(n - 50, n)])
    dst = np.concatenate([rng.integers(0, n, 30_000), rng.integers(0, n // 3, 200_000), np.arange(n - 50, n)])
    w = (1.0 - rng.random(src.size)).astype(np.float32) if weighted else None
    y = gb.random_labels(n, k, 0.8, seed=k + 1)
    dev = torch.device("cuda")
    g = DeviceGraph.from_edges(torch.from_numpy(src).int(), torch.from_numpy(dst).int(),
                               None if w is None else torch.from_numpy(w), n, device=dev, pull=True)
    assert g.n_heavy >= 1
    exp = oracle.serial_embed(src, dst, w, y.labels, n, k)
    lab = torch.from_numpy(y.labels).to(dev)
    emb = Embedder(n, k, dev)
    z = emb.embed(g, lab, variant="pull").cpu().numpy()
    assert emb.reducer_for(g) == "blocks"
    assert rel_err(z, exp) <= TOL
    _force_wide(monkeypatch)
    zw = Embedder(n, k, dev).embed(g, lab, variant="pull").cpu().numpy()
    assert np.array_equal(z.view(np.uint32), zw.view(np.uint32))


@pytest.mark.parametrize("k,weighted", [(1000, False), (1000, True), (301, False), (1001, True), (4096, False)])
def test_wide_k_pull(k, weighted):
    # K > 255 (BASELINE C5 is K = 1000): the fused wide reducer (warp per
    # light row, CTA per heavy row; vector and scalar write-outs for
    # k % 4 == 0 / != 0) against the oracle, and bit-stable
    rng = np.random.default_rng(k + weighted)
    n = 30_011
    hub = np.full(9_000, 11, np.int64)
    src = np.concatenate([hub, rng.integers(0, n, 150_000), np.arange(n - 40, n)])
    dst = np.concatenate([rng.integers(0, n, 9_000), rng.integers(0, n, 150_000), np.arange(n - 40, n)])
    w = (1.0 - rng.random(src.size)).astype(np.float32) if weighted else None
    y = gb.random_labels(n, k, 0.9, seed=k)
    dev = torch.device("cuda")
    g = DeviceGraph.from_edges(torch.from_numpy(src).int(), torch.from_numpy(dst).int(),
                               None if w is None else torch.from_numpy(w), n, device=dev, pull=True)
    assert g.n_heavy >= 1
    exp = oracle.serial_embed(src, dst, w, y.labels, n, k)
    lab = torch.from_numpy(y.labels).to(dev)
    emb = Embedder(n, k, dev)
    assert emb.reducer_for(g) == "wide"
    z = emb.embed(g, lab, variant="pull").cpu().numpy()
    assert rel_err(z, exp) <= TOL
    assert np.array_equal(z.view(np.uint32), emb.embed(g, lab, variant="pull").cpu().numpy().view(np.uint32))


# ---------------------------------------------------------------- signed weights
# The reference accepts any finite weight (graph.py:46-47) and
# states scale equivariance for any constant (SPEC.md:270,
# tests/test_encoder.py:112-119).  With mixed signs a class sum can cancel, so
# the relative bar is taken against the entry's absolute mass
# sum |w| * inv (the oracle run on |w|): |z - ref| <= 1e-4 * mass, and entries
# whose mass is zero are exactly zero.

def signed_err(z, ref, mass):
    z = np.asarray(z, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    mass = np.asarray(mass, dtype=np.float64)
    empty = mass == 0
    assert np.all(z[empty] == 0)
    nz = ~empty
    if not nz.any():
        return 0.0
    return float(np.max(np.abs(z[nz] - ref[nz]) / mass[nz]))


def _signed_case(seed, n, s, k, kind, hub=0):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, s)
    dst = rng.integers(0, n, s)
    if hub:  # rows > 2048 arcs: heavy items (k <= 255) / CTA rows (wide)
        src[:hub] = 3
    if kind == "normal":  # |w| >= 1e-3 keeps the fixed-point gate open (rounding <= 1e-5 of min |w|)
        w = rng.standard_normal(s)
        w = np.where(np.abs(w) < 1e-3, np.copysign(1e-3, w), w).astype(np.float32)
    elif kind == "negative":
        w = -(1.0 - rng.random(s)).astype(np.float32)
    else:  # "cancel": +-1 pairs and small residues, many class sums exactly 0
        w = rng.choice(np.array([1.0, -1.0, 0.5, -0.5], np.float32), s)
    y = gb.random_labels(n, k, 0.9, seed=seed + 1)
    return src, dst, w, y


@pytest.mark.parametrize("variant", ["pull", "push"])
@pytest.mark.parametrize("kind", ["normal", "negative", "cancel"])
@pytest.mark.parametrize("k", [7, 50, 255, 300])
def test_signed_weights(kind, k, variant):
    n, s = 20_011, 250_000
    src, dst, w, y = _signed_case(k * 7 + len(kind), n, s, k, kind, hub=12_000)
    el = gb.EdgeList(n=n, src=src, dst=dst, w=w, directed=True)
    exp = oracle.serial_embed(src, dst, w, y.labels, n, k)
    mass = oracle.serial_embed(src, dst, np.abs(w), y.labels, n, k)
    z = gb.embed_serial(el, y, variant=variant)
    assert signed_err(z, exp, mass) <= TOL, (kind, k, variant)
    if kind == "negative":  # no cancellation: the plain relative bar, and every nonzero entry < 0
        assert rel_err(z, exp) <= TOL
        assert np.all(z[exp != 0] < 0)
    if variant == "pull":
        assert np.array_equal(z.view(np.uint32), gb.embed_serial(el, y, variant="pull").view(np.uint32))


def test_single_negative_arc_exact():
    # the round-1 defect: a class sum of -1 decoded as +4095 * inv
    el = gb.EdgeList(n=3, src=[0, 1], dst=[1, 2], w=[-1.0, 0.5], directed=True)
    y = gb.LabelVector(labels=[1, 1, 2], k=2)
    exp = oracle.serial_embed(el.src, el.dst, el.w, y.labels, 3, 2)
    for variant in ("pull", "push"):
        z = gb.embed_serial(el, y, variant=variant)
        assert np.array_equal(z.astype(np.float64), exp), variant
    assert exp[0, 0] < 0


@pytest.mark.parametrize("c", [-3.5, 3.5, -1.0])
def test_scale_equivariance_signed(c):
    # SPEC.md:270 / test_encoder.py:112-119 (c = 3.5 there), here also for
    # negative c: embed(c * w) == c * embed(w) against the oracle
    n, s, k = 5_003, 80_000, 10
    src, dst, w, y = _signed_case(11, n, s, k, "normal", hub=3_000)
    el = gb.EdgeList(n=n, src=src, dst=dst, w=w, directed=False)
    elc = gb.EdgeList(n=n, src=src, dst=dst, w=(np.float32(c) * w).astype(np.float32), directed=False)
    mass = oracle.serial_embed(src, dst, np.abs(w), y.labels, n, k) * abs(c)
    exp_c = oracle.serial_embed(src, dst, elc.w, y.labels, n, k)
    for variant in ("pull", "push"):
        z = gb.embed_serial(el, y, variant=variant)
        zc = gb.embed_serial(elc, y, variant=variant)
        assert signed_err(zc, exp_c, mass) <= TOL, variant
        assert signed_err(zc, c * z.astype(np.float64), mass) <= 2 * TOL, variant
    if c in (-1.0,):  # negation is exact in the fixed point: bitwise -z
        z = gb.embed_serial(el, y, variant="pull")
        zc = gb.embed_serial(elc, y, variant="pull")
        assert np.array_equal(zc, -z)


@pytest.mark.parametrize("k", [50, 300])
def test_signed_reducers_agree_bitwise(k, monkeypatch):
    # mixed-sign weights through the block reducer, the heavy items (one
    # item and mega rows of several items) and the wide kernel: same bits
    n, s = 70_001, 400_000
    src, dst, w, y = _signed_case(k, n, s, k, "normal", hub=150_000)
    dev = torch.device("cuda")
    g = DeviceGraph.from_edges(torch.from_numpy(src).int(), torch.from_numpy(dst).int(), torch.from_numpy(w), n,
                               device=dev, pull=True)
    g.prepare_hot(k, enable=True)
    assert g.n_heavy >= 1 and g.n_mega >= 1
    lab = torch.from_numpy(y.labels).to(dev)
    emb = Embedder(n, k, dev)
    z = emb.embed(g, lab, variant="pull").cpu().numpy()
    exp = oracle.serial_embed(src, dst, w, y.labels, n, k)
    mass = oracle.serial_embed(src, dst, np.abs(w), y.labels, n, k)
    assert signed_err(z, exp, mass) <= TOL
    _force_wide(monkeypatch)
    zw = Embedder(n, k, dev).embed(g, lab, variant="pull").cpu().numpy()
    assert np.array_equal(z.view(np.uint32), zw.view(np.uint32))


@pytest.mark.parametrize("world", [2, 3])
def test_row_shards_tile_the_full_pull(world):
    # row-range sharding (shard.build_row_shard): each rank's pull over its
    # rows, with the hot tier planned on GLOBAL degrees, run one after the
    # other on this GPU (ranks never wait on each other); the slices tile Z
    from paper_2402_04403_b200 import shard

    scale, s, k = 16, 600_000, 50
    src, dst, w = synth.rmat_edges(scale, s, seed=21, weighted=True)
    n = 1 << scale
    y = synth.uniform_labels(n, k, seed=22)
    exp = oracle.serial_embed(src.cpu().numpy(), dst.cpu().numpy(), w.cpu().numpy(), y.cpu().numpy(), n, k)
    dev = torch.device("cuda")
    shards, bounds = [], []
    for rank in range(world):
        g, lo, hi = shard.build_row_shard(src, dst, w, n, world, rank, k=k)
        g.prepare_hot(k, enable=True)
        assert g.n_hot > 0 and g.global_offsets is None
        shards.append(g)
        bounds.append((lo, hi))
    # the whole graph's fixed-point exponent (bench: one all-reduce) makes
    # the tiled shards bit-identical to the single-GPU pull
    stats = shard.merge_weight_stats(g.weight_stats() for g in shards)
    parts = []
    for g, (lo, hi) in zip(shards, bounds):
        g.adopt_scale(stats)
        emb = Embedder(n, k, dev)
        z = torch.empty((hi - lo, k), dtype=torch.float32, device=dev)
        emb.project(y, g=g)
        parts.append(emb.pull(g, z).cpu().numpy())
    assert bounds[0][0] == 0 and bounds[-1][1] == n
    assert all(bounds[i][1] == bounds[i + 1][0] for i in range(world - 1))
    z_all = np.concatenate(parts)
    assert rel_err(z_all, exp) <= TOL
    single = gb.embed(src, dst, y, n, k, weights=w, directed=True, variant="pull").cpu().numpy()
    assert np.array_equal(z_all, single)


def test_raw_ctypes_binding_without_torch():
    # the C ABI bound with plain ctypes and
    # cuda-python device memory (no torch on the path) reproduces the oracle
    import ctypes

    from cuda.bindings import runtime as rt

    from paper_2402_04403_b200 import _lib

    L = ctypes.CDLL(_lib.LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.gee_last_error.restype = ctypes.c_char_p
    L.gee_build_projection.argtypes = [vp, i64, i32, vp, vp, vp, vp, vp, i64, vp, vp]
    L.gee_embed_coo.argtypes = [vp, vp, vp, i64, vp, i64, vp, i64, i32, vp, ctypes.c_uint32, vp]
    L.gee_label_table_bytes.restype = ctypes.c_size_t

    def check(rc):
        assert rc == 0, L.gee_last_error().decode()

    def dev(a):
        err, p = rt.cudaMalloc(max(a.nbytes, 1))
        assert err == rt.cudaError_t.cudaSuccess
        rt.cudaMemcpy(p, a.ctypes.data, a.nbytes, rt.cudaMemcpyKind.cudaMemcpyHostToDevice)
        return p

    rng = np.random.default_rng(31)
    n, k, s = 5000, 9, 60_000
    src, dst = rng.integers(0, n, s), rng.integers(0, n, s)
    w = (1.0 - rng.random(s)).astype(np.float32)
    y = gb.random_labels(n, k, 0.6, seed=32).labels
    d_src, d_dst, d_w, d_y = dev(src.astype(np.int32)), dev(dst.astype(np.int32)), dev(w), dev(y.astype(np.int32))
    d_counts = rt.cudaMalloc(8 * (k + 1))[1]
    d_inv = rt.cudaMalloc(4 * (k + 1))[1]
    d_tab = rt.cudaMalloc(L.gee_label_table_bytes(n, 0, k))[1]
    d_z = rt.cudaMalloc(4 * n * k)[1]
    try:
        check(L.gee_build_projection(d_y, n, k, d_counts, d_inv, None, d_tab, None, 0, None, None))
        check(L.gee_embed_coo(d_src, d_dst, d_w, s, d_tab, 0, d_inv, n, k, d_z, 1, None))
        z = np.empty((n, k), np.float32)
        rt.cudaMemcpy(z.ctypes.data, d_z, z.nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
        counts = np.empty(k + 1, np.int64)
        rt.cudaMemcpy(counts.ctypes.data, d_counts, counts.nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    finally:
        for p in (d_src, d_dst, d_w, d_y, d_counts, d_inv, d_tab, d_z):
            rt.cudaFree(p)
    assert np.array_equal(counts, np.bincount(y, minlength=k + 1))
    assert rel_err(z, oracle.serial_embed(src, dst, w, y, n, k)) <= TOL


@pytest.mark.parametrize("chunks", [1, 3, 7])
@pytest.mark.parametrize("packed", [True, False])
def test_host_pipeline_matches_resident_pull(chunks, packed):
    # stream.HostPipeline: pinned host graph + labels -> pinned host Z via
    # row chunks on three streams; every chunk's pull sums the same integers
    # as the resident pull, so Z is bit-identical
    from paper_2402_04403_b200.stream import HostPipeline, pinned_like

    scale, s, k = 17, 1_500_000, 50
    src, dst, w = synth.rmat_edges(scale, s, seed=41, weighted=True)
    n = 1 << scale
    y = synth.uniform_labels(n, k, seed=42)
    dev = torch.device("cuda")
    g = DeviceGraph.from_edges(src, dst, w, n, device=dev, pull=True)
    g.prepare_hot(k, enable=True)
    emb = Embedder(n, k, dev)
    emb.project(y, g=g)
    z_ref = emb.pull(g).cpu()
    pipe = HostPipeline(g, k, chunks=chunks, packed=packed)
    assert pipe.n_chunks == chunks and pipe.packed == packed
    h_z = pinned_like((n, k))
    for sparse in (True, False):
        h_z.fill_(float("nan"))
        pipe.run(y.cpu().pin_memory(), h_z, emb, sparse=sparse)
        assert torch.equal(h_z, z_ref), sparse
        if sparse:  # the row-sparse copy-out is smaller than dense Z
            assert 0 < pipe.d2h_bytes < n * k * 4
        else:
            assert pipe.d2h_bytes == n * k * 4
    for dense_every in (1, 2, 3):  # row-sparse chunks mixed with dense ones
        h_z.fill_(float("nan"))
        pipe.run(y.cpu().pin_memory(), h_z, emb, dense_every=dense_every)
        assert torch.equal(h_z, z_ref), dense_every
    exp = oracle.serial_embed(src.cpu().numpy(), dst.cpu().numpy(), w.cpu().numpy(), y.cpu().numpy(), n, k)
    assert rel_err(h_z.numpy(), exp) <= TOL


@pytest.mark.parametrize("rows,k", [(1, 1), (1023, 50), (1024, 64), (5000, 65), (3001, 1000), (0, 7)])
def test_z_compact_round_trip(rows, k):
    # gee_z_compact (device) -> gee_io_expand_rows (host) rebuilds Z bit for
    # bit; the format matches its numpy definition (u64 row masks, packed
    # nonzeros, per-1024-row value offsets); -0.0 counts as a value
    from paper_2402_04403_b200 import _lib
    from paper_2402_04403_b200.formats import io_lib

    rng = np.random.default_rng(rows + k)
    zh = np.where(rng.random((rows, k)) < 0.15, rng.standard_normal((rows, k)), 0.0).astype(np.float32)
    if rows:
        zh[0, 0] = -0.0
        zh[rows // 2] = 0.0
    z = torch.from_numpy(zh).cuda()
    mw = (k + 63) // 64
    nb = int(_lib.lib.gee_zc_blocks(rows))
    mask = torch.empty(max(1, rows * mw), dtype=torch.int64, device="cuda")
    boff = torch.empty(nb + 1, dtype=torch.int64, device="cuda")
    vals = torch.empty(max(1, rows * k), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib.gee_z_compact(_lib.ptr(z), rows, k, _lib.ptr(mask), _lib.ptr(boff), _lib.ptr(vals),
                                      _lib.stream_handle()))
    torch.cuda.synchronize()
    nz = zh.view(np.uint32) != 0
    bits = np.zeros((rows, mw * 64), bool)
    bits[:, :k] = nz
    exp_mask = np.packbits(bits.reshape(rows, mw, 64)[..., ::-1], axis=-1).view(">u8").reshape(rows, mw)
    assert np.array_equal(mask.cpu().numpy()[:rows * mw].view(np.uint64).reshape(rows, mw), exp_mask.astype(np.uint64))
    per_row = nz.sum(1)
    exp_off = np.concatenate([[0], np.cumsum(per_row)])[::1024][:nb]
    assert np.array_equal(boff.cpu().numpy()[:nb], exp_off) and int(boff[nb]) == int(nz.sum())
    assert np.array_equal(vals.cpu().numpy()[:int(nz.sum())].view(np.uint32), zh.view(np.uint32)[nz])
    out = np.full((rows, k), np.nan, np.float32)
    m_h, b_h, v_h = mask.cpu().numpy(), boff.cpu().numpy(), vals.cpu().numpy()
    assert io_lib().gee_io_expand_rows(m_h.ctypes.data, v_h.ctypes.data, b_h.ctypes.data, rows, k,
                                       out.ctypes.data, 3) == 0
    assert np.array_equal(out.view(np.uint32), zh.view(np.uint32))


def test_graph_prep_never_mutates_caller_or_push_arrays():
    # hot encoding and the row sort rewrite the pull targets / weights in
    # place: a caller's CUDA tensors and the push layout must keep theirs
    n, k = 4000, 6
    rng = np.random.default_rng(51)
    el = gb.EdgeList(n=n, src=rng.integers(0, n, 30_000), dst=rng.integers(0, n, 30_000),
                     w=(1.0 - rng.random(30_000)).astype(np.float32), directed=False)
    csr = gb.build_csr(el)
    dev = torch.device("cuda")
    off, tgt, w = (torch.from_numpy(np.asarray(a)).to(dev) for a in (csr.offsets, csr.targets, csr.weights))
    tgt0, w0 = tgt.clone(), w.clone()
    g = DeviceGraph.from_csr(off, tgt, w, n, symmetric=True, device=dev, pull=True, keep_coo=True)
    g.prepare_hot(k, enable=True)
    assert torch.equal(tgt, tgt0) and torch.equal(w, w0)
    assert torch.equal(g.dst, tgt0) and torch.equal(g.w, w0)
    y = gb.random_labels(n, k, 0.8, seed=52)
    yd = torch.from_numpy(y.labels).to(dev)
    emb = Embedder(n, k, dev)
    zp = emb.embed(g, yd, variant="pull").cpu().numpy()
    zq = emb.embed(g, yd, variant="push").cpu().numpy()
    assert rel_err(zp, zq.astype(np.float64)) <= TOL


def _pack_round_trip(off, tgt, w, sentinel):
    from paper_2402_04403_b200 import _lib

    dev = torch.device("cuda")
    off_d = torch.as_tensor(off, dtype=torch.int64, device=dev)
    t_d = torch.as_tensor(tgt, dtype=torch.int32, device=dev)
    w_d = torch.as_tensor(w, dtype=torch.float32, device=dev) if w is not None else None
    arcs = t_d.numel()
    groups = arcs // 8
    u8 = lambda m: torch.empty(max(1, m), dtype=torch.uint8, device=dev)  # noqa: E731
    ctl, pay = u8(groups), u8(4 * arcs)
    wctl, wpay = (u8(groups), u8(4 * arcs)) if w is not None else (None, None)
    nb, nwb = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.lib.gee_pack_targets(_lib.ptr(off_d), off_d.numel() - 1, _lib.ptr(t_d), _lib.ptr(w_d), arcs,
                                         sentinel, _lib.ptr(ctl), _lib.ptr(pay), ctypes.byref(nb), _lib.ptr(wctl),
                                         _lib.ptr(wpay), ctypes.byref(nwb), _lib.stream_handle()), "pack")
    real = t_d != sentinel
    sb = int(_lib.lib.gee_unpack_scratch_bytes(groups))
    scratch = torch.empty(max(1, sb), dtype=torch.uint8, device=dev)
    out_t = torch.full((arcs + 8,), -7, dtype=torch.int32, device=dev)
    out_w = torch.full((arcs + 8,), -7.0, dtype=torch.float32, device=dev) if w is not None else None

    def exact(b, n):  # the bytes a PCIe copy would deliver: exactly n, then junk
        x = torch.full((n + 64,), 0xAB, dtype=torch.uint8, device=dev)
        x[:n] = b[:n]
        return x

    assert int(nb.value) % 4 == 0  # whole u32 words of the bit stream
    pay2 = exact(pay, int(nb.value))
    wpay2 = exact(wpay, int(nwb.value)) if w is not None else None
    # the weight codes as an array, and (when every group shares one) as the
    # chunk's single wctl_uniform byte with no array
    modes = [(wctl, -1)]
    if w is not None and groups and bool((wctl[:groups] == wctl[0]).all()):
        modes.append((None, int(wctl[0])))
    for wc, wu in modes:
        out_t.fill_(-7)
        if out_w is not None:
            out_w.fill_(-7.0)
        _lib.check(_lib.lib.gee_unpack_targets(_lib.ptr(ctl), _lib.ptr(pay2), groups, _lib.ptr(off_d),
                                               off_d.numel() - 1, _lib.ptr(wc), wu, _lib.ptr(wpay2), sentinel,
                                               _lib.ptr(out_t), _lib.ptr(out_w), _lib.ptr(scratch), sb,
                                               _lib.stream_handle()), "unpack")
        torch.cuda.synchronize()
        assert torch.equal(out_t[:arcs], t_d) and bool((out_t[arcs:] == -7).all())
        if w is not None:
            exp_w = torch.where(real, w_d, torch.zeros_like(w_d))
            assert torch.equal(out_w[:arcs].view(torch.int32), exp_w.view(torch.int32))
            assert bool((out_w[arcs:] == -7.0).all())
    if w is not None:
        return int(nb.value), int(nwb.value)
    return int(nb.value), 0


def _padded_rows(degs, rng, sentinel, sort=True, big=False):
    off, tgt, w = [0], [], []
    for d in degs:
        hi = sentinel if big else min(sentinel, 1 << 20)
        row = rng.integers(0, hi, d)
        if sort:
            row = np.sort(row)
        pad = (-d) % 8
        tgt += list(row) + [sentinel] * pad
        w += list(rng.random(d).astype(np.float32) + 0.25) + [0.0] * pad
        off.append(len(tgt))
    return np.array(off), np.array(tgt, dtype=np.int64), np.array(w, dtype=np.float32)


@pytest.mark.parametrize("case", ["mixed", "unsorted", "wide", "single", "empty_rows"])
def test_pack_targets_round_trip(case):
    # gee_pack_targets -> gee_unpack_targets rebuilds the padded targets and
    # weights bit for bit: rows of every length (0, 1, 8, 9, heavy), pads,
    # unsorted rows (deltas wrap mod 2^32) and 4-byte deltas
    rng = np.random.default_rng(len(case))
    sentinel = (1 << 31) - 2 if case == "wide" else 5_000_000
    if case == "single":
        degs = [3]
    elif case == "empty_rows":
        degs = [0, 0, 5, 0, 8, 0, 0, 17, 0]
    else:
        degs = list(rng.integers(0, 40, 3000)) + [0, 1, 8, 9, 7, 16, 5000, 70_000]
        rng.shuffle(degs)
    off, tgt, w = _padded_rows(degs, rng, sentinel, sort=case != "unsorted", big=case == "wide")
    nb, nwb = _pack_round_trip(off, tgt, w, sentinel)
    _pack_round_trip(off, tgt, None, sentinel)
    real = int((tgt != sentinel).sum())
    if case == "mixed":  # sorted rows of 2^20 slots: ~16-bit deltas, well under 3 bytes per real arc
        assert nb < 2.5 * real
    if case == "wide":  # 4-byte deltas at most (32-bit values)
        assert nb <= 4 * real + 4
    # weights of 1 - U[0,1) with 24-bit U: 3 bytes each (groups holding w = 1.0 raw)
    w24 = np.where(tgt != sentinel, 1.0 - rng.integers(0, 1 << 24, tgt.size) / float(1 << 24), 0.0).astype(np.float32)
    _, nwb24 = _pack_round_trip(off, tgt, w24, sentinel)
    assert nwb24 <= 3 * real + real // 8 * 2 + 64


@pytest.mark.parametrize("kind", ["integers", "halves", "mixed_signs", "specials", "tiny", "big"])
def test_pack_weights_lossless(kind):
    # group fixed point is lossless for every f32 pattern: integer and
    # dyadic weights take 1-3 bytes, negatives / -0.0 / denormals / inf /
    # nan / values needing 2^-64 or 4 bytes fall back to raw bits
    rng = np.random.default_rng(len(kind))
    degs = list(rng.integers(0, 30, 2000)) + [1, 8, 9, 300]
    sentinel = 1 << 20
    off, tgt, _ = _padded_rows(degs, rng, sentinel)
    m = tgt.size
    if kind == "integers":
        w = rng.integers(0, 70_000, m).astype(np.float32)
    elif kind == "halves":
        w = (rng.integers(0, 512, m) / 2.0).astype(np.float32)
    elif kind == "mixed_signs":
        w = rng.standard_normal(m).astype(np.float32)
    elif kind == "specials":
        pool = np.array([0.0, -0.0, 1.0, np.inf, -np.inf, np.nan, 1e-45, 3.4e38, 2.0 ** -63, 2.0 ** -64, 0.75],
                        dtype=np.float32)
        w = pool[rng.integers(0, pool.size, m)]
    elif kind == "tiny":
        w = (rng.integers(1, 1 << 20, m) * 2.0 ** -60).astype(np.float32)
    else:
        w = (rng.integers(1, 1 << 24, m).astype(np.float64) * 2.0 ** 30).astype(np.float32)
    w = np.where(tgt != sentinel, w, np.float32(0.0)).astype(np.float32)
    _, nwb = _pack_round_trip(off, tgt, w, sentinel)
    real = int((tgt != sentinel).sum())
    if kind in ("integers", "halves"):
        assert nwb <= 3 * real


def test_pack_targets_many_pads():
    # more than 2^24 pad arcs in one call (C4's chunks hold ~18M): the
    # real-arc index of every group (for the weight copy) stays exact
    rows = 2_500_000
    rng = np.random.default_rng(5)  # (weights: raw or fixed point, per group)
    sentinel = 1 << 27
    tgt = np.full((rows, 8), sentinel, dtype=np.int64)
    tgt[:, 0] = rng.integers(0, sentinel, rows)
    w = np.zeros((rows, 8), dtype=np.float32)
    w[:, 0] = rng.random(rows, dtype=np.float32) + 0.5
    off = np.arange(0, 8 * rows + 1, 8)
    _pack_round_trip(off, tgt.ravel(), w.ravel(), sentinel)


def test_pack_targets_rejects_unpadded():
    from paper_2402_04403_b200 import _lib

    dev = torch.device("cuda")
    off = torch.tensor([0, 16], dtype=torch.int64, device=dev)
    t = torch.tensor([1, 2, 3, 9, 9, 9, 9, 9, 9, 9, 9, 9, 9, 9, 9, 9], dtype=torch.int32, device=dev)  # 13 pads
    ctl = torch.empty(2, dtype=torch.uint8, device=dev)
    pay = torch.empty(64, dtype=torch.uint8, device=dev)
    nb = ctypes.c_int64()
    rc = _lib.lib.gee_pack_targets(_lib.ptr(off), 1, _lib.ptr(t), None, 16, 9, _lib.ptr(ctl), _lib.ptr(pay),
                                   ctypes.byref(nb), None, None, None, _lib.stream_handle())
    assert rc != 0 and b"padded layout" in _lib.lib.gee_last_error()


@pytest.mark.parametrize("head", [-1, 40000, 0])
@pytest.mark.parametrize("k", [5, 20, 50, 63, 64, 200])
def test_gather_labels_heads(k, head):
    # gee_gather_labels equals a plain gather for every kernel variant: the
    # shared-memory head packed 8 / 6 / 5 / 4 labels per word by k (full and
    # partial heads) and plain contiguous lookups; skewed slots hit the head,
    # the hot tier and the cold tier; ragged lengths exercise the tails
    from paper_2402_04403_b200 import _lib

    gen = torch.Generator(device="cuda").manual_seed(k)
    n_hot, n = 300_000, 2_000_000
    table = torch.randint(0, k + 1, (n_hot + n + 1,), dtype=torch.uint8, device="cuda", generator=gen)
    for arcs in (5, 512 * 148 * 32 + 77, 3_000_001):
        u = torch.rand(arcs, device="cuda", generator=gen)
        t = torch.where(u < 0.5, (u * 200_000).long(), torch.where(
            u < 0.75, (u * n_hot).long() % n_hot, torch.randint(0, n_hot + n + 1, (arcs,), device="cuda",
                                                                 generator=gen))).int()
        cls = torch.full((arcs + 16,), 255, dtype=torch.uint8, device="cuda")
        _lib.check(_lib.lib.gee_gather_labels_head(_lib.ptr(t), arcs, _lib.ptr(table), n_hot, k, head,
                                                   _lib.ptr(cls), _lib.stream_handle()), "gee_gather_labels_head")
        torch.cuda.synchronize()
        assert torch.equal(cls[:arcs], table[t.long()]), arcs
        assert bool((cls[arcs:] == 255).all()), arcs


@pytest.mark.parametrize("k", [50, 300, 70_000])
def test_projection_compact_hot_tier(k):
    # gee_build_projection_hotc (bitmap + prefix + ranks in vertex order)
    # writes the same label table and counts as the hot_rank form, for u8,
    # u16 and int32 tables, with a ragged n (not a multiple of 4 or 32)
    from paper_2402_04403_b200 import _lib

    n = 1_000_003
    dev = torch.device("cuda")
    gen = torch.Generator(device="cuda").manual_seed(k)
    hot = torch.rand(n, device=dev, generator=gen) < 0.2
    n_hot = int(hot.sum())
    hot_rank = torch.full((n,), -1, dtype=torch.int32, device=dev)
    hot_rank[hot] = torch.randperm(n_hot, device=dev, generator=gen).int()
    labels = torch.randint(0, k + 1, (n,), dtype=torch.int32, device=dev, generator=gen)
    g = DeviceGraph(n, 0, dev)
    g.hot_rank = hot_rank
    g.compact_hot()
    lb = int(_lib.lib.gee_label_bytes(k))
    tb = int(_lib.lib.gee_label_table_bytes(n, n_hot, k))
    out = []
    for compact in (False, True):
        table = torch.full((tb,), 0xEE, dtype=torch.uint8, device=dev)
        counts = torch.zeros(k + 1, dtype=torch.int64, device=dev)
        if compact:
            rc = _lib.lib.gee_build_projection_hotc(_lib.ptr(labels), n, k, _lib.ptr(counts), None, None,
                                                    _lib.ptr(table), _lib.ptr(g.hot_bits), _lib.ptr(g.hot_pref),
                                                    _lib.ptr(g.hot_list), n_hot, None, _lib.stream_handle())
        else:
            rc = _lib.lib.gee_build_projection(_lib.ptr(labels), n, k, _lib.ptr(counts), None, None,
                                               _lib.ptr(table), _lib.ptr(hot_rank), n_hot, None,
                                               _lib.stream_handle())
        assert rc == 0, _lib.lib.gee_last_error()
        torch.cuda.synchronize()
        out.append((table.cpu().numpy(), counts.cpu().numpy()))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    assert np.array_equal(out[1][1], np.bincount(labels.cpu().numpy(), minlength=k + 1))
    # the hot prefix holds each hot vertex's label at its rank
    tab = out[1][0][:(n_hot + n + 1) * lb].view({1: np.uint8, 2: np.uint16, 4: np.int32}[lb])
    hv = np.flatnonzero(hot.cpu().numpy())
    assert np.array_equal(tab[hot_rank.cpu().numpy()[hv]], labels.cpu().numpy()[hv])
    assert np.array_equal(tab[n_hot:n_hot + n], labels.cpu().numpy())


@pytest.mark.parametrize("k", [5, 300])
def test_projection_counts_out_of_range_labels(k):
    # labels outside [0, k] (LabelVector rejects them, labeling.py:24-29) are
    # reported through `bad`, left out of the counts and stored as 0
    from paper_2402_04403_b200 import _lib

    dev = torch.device("cuda")
    lab = torch.tensor([1, -1, k, k + 1, 0, 2**31 - 1, 3, -(2**31)] * 1001, dtype=torch.int32, device=dev)
    n = lab.numel()
    tb = int(_lib.lib.gee_label_table_bytes(n, 0, k))
    table = torch.full((tb,), 0xEE, dtype=torch.uint8, device=dev)
    counts = torch.zeros(k + 1, dtype=torch.int64, device=dev)
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    rc = _lib.lib.gee_build_projection(_lib.ptr(lab), n, k, _lib.ptr(counts), None, None, _lib.ptr(table), None, 0,
                                       _lib.ptr(bad), _lib.stream_handle())
    assert rc == 0
    torch.cuda.synchronize()
    assert int(bad.item()) == 4 * 1001
    exp = np.zeros(k + 1, dtype=np.int64)
    exp[[1, k, 0, 3]] += 1001
    assert np.array_equal(counts.cpu().numpy(), exp)
    lb = int(_lib.lib.gee_label_bytes(k))
    tab = table.cpu().numpy()[:(n + 1) * lb].view({1: np.uint8, 2: np.uint16}[lb])
    want = np.where((lab.cpu().numpy() >= 0) & (lab.cpu().numpy() <= k), lab.cpu().numpy(), 0)
    assert np.array_equal(tab[:n], want) and tab[n] == 0


@pytest.mark.parametrize("k,labeled", [(100, 0.1), (5, 1.0)])
def test_host_pipeline_unit_weights(k, labeled):
    # the streamed pass on an unweighted graph (packed targets, no weight
    # streams; C3-like 10% labeled K=100 and a small-K table): Z equals the
    # resident pull bit for bit, and the oracle within tolerance
    from paper_2402_04403_b200.stream import HostPipeline, pinned_like

    scale, s = 16, 600_000
    n = 1 << scale
    src, dst, _ = synth.rmat_edges(scale, s, seed=k, weighted=False)
    y = torch.from_numpy(gb.random_labels(n, k, labeled, seed=k).labels).cuda()
    dev = torch.device("cuda")
    g = DeviceGraph.from_edges(src, dst, None, n, device=dev, pull=True)
    g.prepare_hot(k, enable=True)
    emb = Embedder(n, k, dev)
    emb.project(y, g=g)
    z_ref = emb.pull(g).cpu()
    pipe = HostPipeline(g, k, chunks=3)
    assert pipe.packed and not pipe.weighted
    h_z = pinned_like((n, k))
    h_z.fill_(float("nan"))
    pipe.run(y.cpu().pin_memory(), h_z, emb)
    assert torch.equal(h_z, z_ref)
    exp = oracle.serial_embed(src.cpu().numpy(), dst.cpu().numpy(), None, y.cpu().numpy(), n, k)
    assert rel_err(h_z.numpy(), exp) <= TOL


# ---------------------------------------------------------------- projection= / variant policy
def test_projection_is_honoured(golden):
    # a caller-supplied ProjectionMatrix is used, not recomputed
    # (encoder.py:116 embed_serial: y.labels with projection.row_value;
    # encoder.py:155,180-181 embed_parallel: projection.label / row_value)
    c = case(golden, "rand4")
    el, y = _el(c), _y(c)
    k = y.k
    proj = gb.build_projection(y)
    scale = np.arange(1, k + 2, dtype=np.float64)  # class c scaled by c + 1
    custom = gb.ProjectionMatrix(n=proj.n, k=k, row_value=proj.row_value * scale[proj.label], label=proj.label)
    exp = c["z_serial"] * scale[1:]
    for variant in ("pull", "push"):
        assert rel_err(gb.embed_serial(el, y, projection=custom, variant=variant), exp) <= TOL, variant
        g = gb.build_csr(el)
        assert rel_err(gb.embed_parallel(g, y, projection=custom, variant=variant), exp) <= TOL, variant
    # embed_parallel reads the projection's labels, not y's
    shifted = np.where(proj.label > 0, proj.label % k + 1, 0).astype(np.int32)
    alt = gb.ProjectionMatrix(n=proj.n, k=k, row_value=proj.row_value, label=shifted)
    z_alt = gb.embed_parallel(gb.build_csr(el), y, projection=alt, variant="pull")
    exp_alt = oracle.serial_embed(el.src, el.dst, el.w, shifted, el.n, k)
    # same labels as `shifted`, but each class keeps the value of the class it came from
    _, inv_old, _ = oracle.projection(y.labels, k)
    _, inv_new, _ = oracle.projection(shifted, k)
    old_of_new = np.zeros(k + 1)
    old_of_new[shifted[y.labels > 0]] = inv_old[y.labels[y.labels > 0]]
    ratio = np.divide(old_of_new, inv_new, out=np.zeros(k + 1), where=inv_new > 0)
    assert rel_err(z_alt, exp_alt * ratio[1:]) <= TOL


def test_projection_per_node_values_rejected(golden):
    c = case(golden, "rand4")
    y = _y(c)
    proj = gb.build_projection(y)
    rv = proj.row_value.copy()
    i = int(np.nonzero(proj.label)[0][0])
    rv[i] *= 1.5
    bad = gb.ProjectionMatrix(n=proj.n, k=proj.k, row_value=rv, label=proj.label)
    with pytest.raises(gb.ValidationError, match="constant within each class"):
        gb.embed_serial(_el(c), y, projection=bad)
    with pytest.raises(gb.ValidationError):
        gb.embed_serial(_el(c), y, projection=gb.ProjectionMatrix(n=proj.n + 1, k=proj.k, row_value=rv,
                                                                    label=proj.label))


def test_variant_policy_and_gate_warning(golden, caplog):
    from paper_2402_04403_b200 import encoder

    c = case(golden, "rand4")
    el, y = _el(c), _y(c)
    gb.embed_serial(el, y)
    assert encoder.last_pass()["variant"] == "pull"
    g = gb.build_csr(el)
    gb.embed_parallel(g, y)
    assert encoder.last_pass()["variant"] == "push"  # small graph: measured table
    gb.embed_parallel(g, y, atomics=False)
    assert encoder.last_pass()["variant"] == "pull"
    # weights spanning 1e-9 .. 1: the fixed point refuses, auto falls back loudly
    w = np.ones(el.s, np.float32)
    w[0] = 1e-9
    wide = gb.EdgeList(n=el.n, src=el.src, dst=el.dst, w=w, directed=el.directed)
    with caplog.at_level("WARNING"):
        z = gb.embed_serial(wide, y)
    assert encoder.last_pass()["variant"] == "push" and "gate" in encoder.last_pass()["reason"]
    assert any("push variant" in r.getMessage() for r in caplog.records)
    exp = oracle.serial_embed(el.src, el.dst, w, y.labels, el.n, y.k)
    assert rel_err(z, exp) <= TOL
    with pytest.raises(gb.ValidationError, match="push"):
        gb.embed_serial(wide, y, variant="pull")


@pytest.mark.parametrize("variant", ["pull", "push"])
def test_captured_pass_replays_on_new_labels(variant):
    # one edge pass recorded as a CUDA graph (Embedder.capture): replaying
    # it after the labels change gives the eager result for the new labels
    scale, s, k = 14, 200_000, 5
    n = 1 << scale
    src, dst, w = synth.rmat_edges(scale, s, seed=61, weighted=True)
    g = DeviceGraph.from_edges(src, dst, w, n, pull=True, keep_coo=True)
    emb = Embedder(n, k)
    y = synth.uniform_labels(n, k, seed=61)
    z = torch.empty((n, k), dtype=torch.float32, device="cuda")
    graph = emb.capture(g, y, z, variant=variant)
    for seed in (62, 63):
        y.copy_(synth.uniform_labels(n, k, seed=seed))
        z.fill_(float("nan"))
        graph.replay()
        torch.cuda.synchronize()
        ref = Embedder(n, k).embed(g, y, variant=variant)
        if variant == "pull":
            assert torch.equal(z, ref)
        else:
            assert rel_err(z.cpu().numpy(), ref.cpu().numpy().astype(np.float64)) <= TOL
