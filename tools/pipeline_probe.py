"""Chunked gather -> block-reduce on the resident C4 graph: does the class
stream stay in L2 when each row chunk is reduced right after its gather, and
do gather(c+1) and blocks(c) overlap on two streams?  (heavy rows excluded:
they are reduced by their own pass.)  Dev tool.

    python tools/pipeline_probe.py [chunks ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_04403_b200 import synth  # noqa: E402
from paper_2402_04403_b200._lib import check, lib  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph, Embedder  # noqa: E402
from paper_2402_04403_b200.shard import plan_rows  # noqa: E402

chunk_list = [int(a) for a in sys.argv[1:]] or [8, 32, 128]
src, dst, w, y, n, k, _ = synth.make_config(4)
g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
del src, dst, w
g.prepare_hot(k)
emb = Embedder(n, k, g.device)
emb.project(y, g=g)
z = emb.pull(g)
torch.cuda.synchronize()
off_h = g.offsets.cpu().numpy()
P = lambda t, byte_off=0: ctypes.c_void_p(t.data_ptr() + byte_off)  # noqa: E731
import ctypes  # noqa: E402

s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def gather(a0, a1, st):
    a0 &= ~15
    a1 = min(g.arcs, (a1 + 15) & ~15)
    check(lib.gee_gather_labels(P(g.targets, 4 * a0), a1 - a0, P(emb.table), g.n_hot, k, P(emb.cls, a0),
                                st.cuda_stream), "gather")


def blocks(lo, hi, st):
    check(lib.gee_reduce_blocks_pad8(P(g.offsets, 8 * lo), hi - lo, P(emb.cls), P(g.weights), g.scale_exp,
                                     P(emb.inv64), k, g.HEAVY_ARCS, P(z, 4 * k * lo), st.cuda_stream), "blocks")


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


cur = torch.cuda.current_stream()
base = timed(lambda: (gather(0, g.arcs, cur), blocks(0, g.n, cur)))
ga = timed(lambda: gather(0, g.arcs, cur))
print(f"whole: gather {ga:.2f} ms, gather+blocks {base:.2f} ms", flush=True)
for C in chunk_list:
    bnd = plan_rows(off_h, C, k, True)
    bnd[1:-1] = (bnd[1:-1] // 32) * 32  # block-aligned (z rows 16-byte aligned)
    spans = [(int(bnd[c]), int(bnd[c + 1]), int(off_h[bnd[c]]), int(off_h[bnd[c + 1]])) for c in range(C)]

    def seq():
        for lo, hi, a0, a1 in spans:
            gather(a0, a1, cur)
            blocks(lo, hi, cur)

    def pipe():
        ev_g = [torch.cuda.Event() for _ in spans]
        ev_b = [torch.cuda.Event() for _ in spans]
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        for i, (lo, hi, a0, a1) in enumerate(spans):
            if i >= 2:
                s1.wait_event(ev_b[i - 2])  # at most one chunk ahead (its cls stays hot)
            gather(a0, a1, s1)
            ev_g[i].record(s1)
            s2.wait_event(ev_g[i])
            blocks(lo, hi, s2)
            ev_b[i].record(s2)
        cur.wait_stream(s2)

    t_seq = timed(seq)
    t_pipe = timed(pipe)
    print(f"chunks {C}: sequential {t_seq:.2f} ms  two-stream {t_pipe:.2f} ms", flush=True)
