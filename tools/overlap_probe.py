"""Can the gather and the block reduction overlap on one GPU?  Times each
alone and both concurrently on two streams (same prepared C4 graph; the
concurrent run writes separate outputs).  Dev tool."""
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
emb = Embedder(n, k, g.device)
emb.project(y, g=g)
z = emb.pull(g)
cls2 = torch.empty_like(emb.cls)
z2 = torch.empty_like(z)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def gather(cls, st):
    check(lib.gee_gather_labels(ptr(g.targets), g.arcs, ptr(emb.table), g.n_hot, k, ptr(cls), st.cuda_stream), "g")


def blocks(zz, st):
    check(lib.gee_reduce_blocks_pad8(ptr(g.offsets), g.n, ptr(emb.cls), ptr(g.weights), g.scale_exp, ptr(emb.inv64),
                                     k, g.HEAVY_ARCS, ptr(zz), st.cuda_stream), "b")


def timed(fn, reps=3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


for _ in range(2):
    ga = timed(lambda: gather(cls2, s1))
    bl = timed(lambda: blocks(z2, s2))
    both = timed(lambda: (gather(cls2, s1), blocks(z2, s2)))
print(f"gather {ga:.2f} ms  blocks {bl:.2f} ms  sum {ga + bl:.2f}  concurrent {both:.2f} ms "
      "")
