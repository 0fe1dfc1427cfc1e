# How fast can the C4 label lookups go in isolation?  (torch gather on the real
# hot-encoded targets; diagnostic only)
import sys, time, torch
sys.path.insert(0, '.')
from paper_2402_04403_b200 import synth
from paper_2402_04403_b200.device import DeviceGraph, Embedder
src, dst, w, y, n, k, directed = synth.make_config(4)
g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
del src, dst, w
torch.cuda.empty_cache()
emb = Embedder(n, k)
g.prepare_hot(k)
emb.project(y, g=g)
tab = emb.table
tgt = g.targets
print("arcs", tgt.numel(), "n_hot", g.n_hot, "table MB", tab.numel() / 1e6)
hot = (tgt < g.n_hot)
print("hot fraction", hot.float().mean().item(), "smem(<93K) fraction", (tgt < 92976).float().mean().item())
def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
chunk = 1 << 29
def gather_all():
    s = 0
    for i in range(0, tgt.numel(), chunk):
        s = s + tab[tgt[i:i + chunk].long()].sum(dtype=torch.int64)
    return s
def stream_only():
    s = 0
    for i in range(0, tgt.numel(), chunk):
        s = s + tgt[i:i + chunk].long().sum()
    return s
#print("stream targets only ms", timeit(stream_only))
#print("gather all ms", timeit(gather_all))
t2 = torch.where(hot, tgt, torch.zeros_like(tgt))
def gather_hot():
    s = 0
    for i in range(0, t2.numel(), chunk):
        s = s + tab[t2[i:i + chunk].long()].sum(dtype=torch.int64)
    return s
#print("gather hot-only (cold->slot0) ms", timeit(gather_hot))
from paper_2402_04403_b200 import _lib
cls = torch.empty(tgt.numel(), dtype=torch.uint8, device="cuda")
def mine():
    _lib.check(_lib.lib.gee_gather_labels(_lib.ptr(tgt), tgt.numel(), _lib.ptr(tab), g.n_hot, k, _lib.ptr(cls), _lib.stream_handle()))
print("gee_gather_labels ms", timeit(mine))
ref = tab[tgt[:1000000].long()]
print("check", bool((cls[:1000000] == ref).all()))
def mine_cold():
    _lib.check(_lib.lib.gee_gather_labels(_lib.ptr(tgt), tgt.numel(), _lib.ptr(tab), 0, k, _lib.ptr(cls), _lib.stream_handle()))
print("gee_gather_labels (no smem head) ms", timeit(mine_cold))
