"""Dev tool: with the tile-major heavy region, can the light rows' gather
(L1 -> L2 request-bound) overlap the heavy reducer (shared-atomic-bound)?
Times each alone and both on two streams, C4."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_04403_b200 import synth  # noqa: E402
from paper_2402_04403_b200._lib import check, lib, ptr  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph, Embedder  # noqa: E402

src, dst, w, y, n, k, _ = synth.make_config(4)
g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
del src, dst, w
g.prepare_hot(k)
g.tile_heavy(max_tiles=21)
emb = Embedder(n, k, g.device)
emb.project(y, g=g)
z = emb.pull(g)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def light(st):
    check(lib.gee_gather_labels(ptr(g.targets), g.light_arcs, ptr(emb.table), g.n_hot, k, ptr(emb.cls),
                                st.cuda_stream), "g")


def heavy(st):
    check(lib.gee_reduce_heavy(ptr(emb.cls), ptr(g.weights), g.arcs, g.scale_exp, ptr(emb.inv64), k,
                               ptr(g.item_first), ptr(g.item_end), ptr(g.item_row), ptr(g.item_slot), g.n_items,
                               ptr(g.mega_rows), g.n_mega, ptr(emb.mega_acc) if g.n_mega else None,
                               ptr(emb.counter), ptr(z), st.cuda_stream), "h")


def timed(fn, reps=5):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


for _ in range(2):
    ga = timed(lambda: light(s1))
    hv = timed(lambda: heavy(s2))
    both = timed(lambda: (light(s1), heavy(s2)))
    both2 = timed(lambda: (heavy(s2), light(s1)))
    print(f"light gather {ga:.2f} ms  heavy {hv:.2f} ms  sum {ga + hv:.2f}  concurrent (gather first) {both:.2f} ms  "
          f"(heavy first) {both2:.2f} ms", flush=True)
