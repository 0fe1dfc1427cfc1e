"""Dev tool: does an L2 persisting access-policy window over the hot tier of
the label table (set-aside L2) speed up the L2-path gathers?  C4, tile
layout: light rows' gather and the heavy tail, with and without the window."""
import json
import sys

import torch
from cuda.bindings import runtime as rt

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
g.tile_heavy()
emb = Embedder(n, k)
emb.project(y, g=g)
z = emb.pull(g)
st = _lib.stream_handle()
stream = torch.cuda.current_stream().cuda_stream


def light():
    check(lib.gee_gather_labels_head(ptr(g.targets), g.light_arcs, ptr(emb.table), g.n_hot, k, 131072, ptr(emb.cls), st), "g")


def tail():
    check(lib.gee_gather_scatter(ptr(g.targets), g.light_arcs, g.l2_arcs, g.light_arcs, ptr(g.group_dst), ptr(emb.table),
                                 k, ptr(emb.cls), st), "t")


def step():
    emb.project(y, validate=False, g=g)
    emb.pull(g, z)


out = {"base": {"light": timeit(light), "tail": timeit(tail), "step": timeit(step)}}
print(json.dumps(out), flush=True)
err, prop = rt.cudaGetDeviceProperties(0)
out["persistingL2CacheMaxSize"] = int(prop.persistingL2CacheMaxSize)
out["accessPolicyMaxWindowSize"] = int(prop.accessPolicyMaxWindowSize)
for set_aside_mb, win_mb in ((32, 16), (64, 16), (64, 48), (96, 64)):
    (err,) = rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, set_aside_mb << 20)
    attr = rt.cudaStreamAttrValue()
    attr.accessPolicyWindow.base_ptr = emb.table.data_ptr()
    attr.accessPolicyWindow.num_bytes = min(win_mb << 20, emb.table.numel())
    attr.accessPolicyWindow.hitRatio = 1.0
    attr.accessPolicyWindow.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
    attr.accessPolicyWindow.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
    (err2,) = rt.cudaStreamSetAttribute(stream, rt.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow, attr)
    key = f"set_aside_{set_aside_mb}MB_window_{win_mb}MB"
    out[key] = {"rc": [int(err), int(err2)], "light": timeit(light), "tail": timeit(tail), "step": timeit(step)}
    print(json.dumps({key: out[key]}), flush=True)
rt.cudaCtxResetPersistingL2Cache()
print(json.dumps(out))
