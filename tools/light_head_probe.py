"""Dev tool: shared-memory head size of the L2-path gather once the heavy
rows live in the tile-major region (light rows only), C4."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2402_04403_b200 import _lib, synth  # noqa: E402
from paper_2402_04403_b200._lib import check, lib, ptr  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph, Embedder  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


src, dst, w, y, n, k, directed = synth.make_config(4)
g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
del src, dst, w
g.prepare_hot(k)
g.tile_heavy(max_tiles=21)
emb = Embedder(n, k)
emb.project(y, g=g)
emb.pull(g)
st = _lib.stream_handle()
out = {"light_arcs": g.light_arcs, "head_ms": {}}
for head in (0, 65536, 98304, 114688, 131072, 147456, 163840):
    def gather():
        check(lib.gee_gather_labels_head(ptr(g.targets), g.light_arcs, ptr(emb.table), g.n_hot, k, head, ptr(emb.cls),
                                         st), "gather")
    out["head_ms"][head] = round(timeit(gather), 3)
out["tail_ms"] = round(timeit(lambda: check(lib.gee_gather_scatter(
    ptr(g.targets), g.light_arcs, g.l2_arcs, g.light_arcs, ptr(g.group_dst), ptr(emb.table), k, ptr(emb.cls), st), "t")), 3)
out["tiles_ms"] = round(timeit(lambda: check(lib.gee_gather_tiles(
    ptr(g.targets), ptr(g.tile_start), g.n_tiles, g.light_arcs, ptr(g.group_dst), ptr(emb.table), g.n_hot + n + 1,
    g.tile_slots, k, ptr(emb.cls), st), "t")), 3)
out["tail_arcs"] = g.l2_arcs - g.light_arcs
out["tile_arcs"] = g.arcs - g.l2_arcs
print(json.dumps(out))
