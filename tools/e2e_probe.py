"""Where does the e2e (HostPipeline) time go on C4?  copy-in alone, copy-in +
compute, full run (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_04403_b200 import synth  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph, Embedder  # noqa: E402
from paper_2402_04403_b200.stream import HostPipeline, pinned_like  # noqa: E402

src, dst, w, y, n, k, _ = synth.make_config(4)
g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
del src, dst, w
torch.cuda.empty_cache()
g.prepare_hot(k)
emb = Embedder(n, k)
emb.project(y, g=g)
chunks = int(os.environ.get("CHUNKS", "16"))
pipe = HostPipeline(g, k, chunks=chunks)
h_y = y.cpu().pin_memory()
h_z = pinned_like((n, k))
pipe.run(h_y, h_z, emb)
torch.cuda.synchronize()


def copy_in():
    for i, v in enumerate(pipe.views):
        b = i & 1
        lo, hi, a0, a1 = v.span
        with torch.cuda.stream(pipe.s_in):
            pipe.d_off[b][:hi - lo + 1].copy_(pipe.h_off[i], non_blocking=True)
            pipe.d_ctl[b][:pipe.h_ctl[i].numel()].copy_(pipe.h_ctl[i], non_blocking=True)
            pipe.d_pay[b][:pipe.h_pay[i].numel()].copy_(pipe.h_pay[i], non_blocking=True)
            pipe.d_wr[b][:pipe.h_wr[i].numel()].copy_(pipe.h_wr[i], non_blocking=True)
    pipe.s_in.synchronize()


def timed(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


hb = pipe.h2d_bytes(h_y)
ms = timed(copy_in)
print(f"copy-in only: {ms:.1f} ms  ({hb / ms / 1e6:.1f} GB/s over {hb / 1e9:.2f} GB)")
dz = torch.empty(n * k // chunks + 1, dtype=torch.float32, device="cuda")
big = torch.empty(int(3.6e9) // 4, dtype=torch.float32).pin_memory()
dbig = torch.empty_like(big, device="cuda")
def both():
    with torch.cuda.stream(pipe.s_out):
        big.copy_(dbig, non_blocking=True)
    copy_in()
    pipe.s_out.synchronize()
print(f"copy-in + 3.6 GB D2H concurrently: {timed(both):.1f} ms")
print(f"full run sparse: {timed(lambda: pipe.run(h_y, h_z, emb)):.1f} ms")
t0 = time.perf_counter()
h_z.fill_(0.0)
print(f"host fill of Z ({h_z.numel() * 4 / 1e9:.1f} GB): {(time.perf_counter() - t0) * 1e3:.1f} ms")
import threading  # noqa: E402


def expand_all():
    # every chunk's expansion from slot 0's compacted rows (host write rate)
    from paper_2402_04403_b200.formats import io_lib
    import ctypes
    from paper_2402_04403_b200 import _lib
    lo, hi, _, _ = pipe.views[0].span
    for i in range(len(pipe.views)):
        io_lib().gee_io_expand_rows(_lib.ptr(pipe.hm[0]), _lib.ptr(pipe.hv[0]), _lib.ptr(pipe.hb[0]), hi - lo, k,
                                    ctypes.c_void_p(h_z.data_ptr()), 0)


print(f"expand x{len(pipe.views)} chunks alone: {timed(expand_all):.1f} ms")


def copy_in_with_fill():
    t = threading.Thread(target=lambda: h_z.fill_(0.0))
    t.start()
    copy_in()
    t.join()


print(f"copy-in + host fill of Z concurrently: {timed(copy_in_with_fill):.1f} ms")


def copy_in_with_expand():
    t = threading.Thread(target=expand_all)
    t.start()
    copy_in()
    t.join()


print(f"copy-in + expand concurrently: {timed(copy_in_with_expand):.1f} ms")
