"""Dev tool: can a cudaMemsetAsync of the whole Z (26.8 GB on C4) hide behind
the light rows' gather (L1 -> L2 request-bound, DRAM at ~40%)?  If so the
block reducer could skip its zero fill.  Times each alone and both on two
streams; also a torch fill kernel for comparison."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

from paper_2402_04403_b200 import synth  # noqa: E402
from paper_2402_04403_b200._lib import check, lib, ptr  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph, Embedder  # noqa: E402

src, dst, w, y, n, k, _ = synth.make_config(4)
g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
del src, dst, w
g.prepare_hot(k)
g.tile_heavy()
emb = Embedder(n, k, g.device)
emb.project(y, g=g)
z = emb.pull(g)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def light(st):
    check(lib.gee_gather_labels_head(ptr(g.targets), g.light_arcs, ptr(emb.table), g.n_hot, k, 131072, ptr(emb.cls),
                                     st.cuda_stream), "g")


def tiles(st):
    check(lib.gee_gather_scatter(ptr(g.targets), g.light_arcs, g.l2_arcs, g.light_arcs, ptr(g.group_dst),
                                 ptr(emb.table), k, ptr(emb.cls), st.cuda_stream), "t")
    check(lib.gee_gather_tiles(ptr(g.targets), ptr(g.tile_start), g.n_tiles, g.light_arcs, ptr(g.group_dst),
                               ptr(emb.table), g.n_hot + n + 1, g.tile_slots, k, ptr(emb.cls), st.cuda_stream), "t")


def memset(st):
    (err,) = rt.cudaMemsetAsync(z.data_ptr(), 0, z.numel() * 4, st.cuda_stream)
    assert int(err) == 0, err


def fill(st):
    with torch.cuda.stream(st):
        z.zero_()


def timed(fn, reps=5):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


for _ in range(2):
    ga, ti, ms, fl = timed(lambda: light(s1)), timed(lambda: tiles(s1)), timed(lambda: memset(s2)), timed(lambda: fill(s2))
    print(f"light gather {ga:.2f}  tail+tiles {ti:.2f}  cudaMemsetAsync(Z) {ms:.2f}  torch fill {fl:.2f} ms", flush=True)
    print(f"  gather || memset {timed(lambda: (light(s1), memset(s2))):.2f}   memset first {timed(lambda: (memset(s2), light(s1))):.2f}"
          f"   gather || torch fill {timed(lambda: (light(s1), fill(s2))):.2f}"
          f"   (gather + tiles) || memset {timed(lambda: (light(s1), tiles(s1), memset(s2))):.2f}", flush=True)
