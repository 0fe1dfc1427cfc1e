"""Runtime-parameter sweep on C4 (dev tool): shared-memory head size of the
gather, heavy-row threshold and heavy work-item size.  Times each variant's
kernels with CUDA events (10 reps) and checks the class stream / Z bits
against the default."""
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
out = {"head": {}, "heavy": {}}
g = DeviceGraph.from_edges(src, dst, w, n, pull=True, keep_coo=True)
g.prepare_hot(k)
emb = Embedder(n, k)
emb.project(y, g=g)
z_ref = emb.pull(g).clone()
ref_cls = emb.cls[:g.arcs].clone()
st = _lib.stream_handle()
for head in (0, 65536, 81920, 98304, 114688, 131072):
    def gather():
        check(lib.gee_gather_labels_head(ptr(g.targets), g.arcs, ptr(emb.table), g.n_hot, k, head, ptr(emb.cls), st),
              "gather")
    out["head"][head] = {"ms": timeit(gather), "same": bool(torch.equal(emb.cls[:g.arcs], ref_cls))}
print(json.dumps(out), flush=True)
src_h = (g.src, g.dst, g.w)
del g, emb
torch.cuda.empty_cache()
for heavy_arcs, item in ((2048, 65536), (2048, 32768), (2048, 131072), (1024, 65536), (1536, 65536)):
    DeviceGraph.HEAVY_ARCS, DeviceGraph.HEAVY_ITEM_ARCS = heavy_arcs, item
    g = DeviceGraph.from_edges(*src_h, n, pull=True)
    g.prepare_hot(k)
    emb = Embedder(n, k)
    emb.project(y, g=g)
    z = emb.pull(g)
    ms = timeit(lambda: (emb.project(y, validate=False, g=g), emb.pull(g, z)))
    out["heavy"][f"{heavy_arcs}/{item}"] = {"step_ms": ms, "same": bool(torch.equal(z, z_ref)),
                                           "n_heavy": g.n_heavy, "items": g.n_items}
    del g, emb, z
    torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)
