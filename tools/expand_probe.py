"""Host-side expansion throughput of the row-sparse Z (dev tool): C4 through
prepare(residency='device'), then gee_io_expand_rows on one chunk's host slot,
timed alone; and the copy-out alone."""
import ctypes
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2402_04403_b200 import CsrGraph, EdgeList, LabelVector, build_csr, embed_parallel, prepare, synth  # noqa
from paper_2402_04403_b200 import _lib  # noqa: E402
from paper_2402_04403_b200.formats import io_lib  # noqa: E402

src, dst, w, y, n, k, directed = synth.make_config(4)
c = build_csr(EdgeList(n=n, src=src, dst=dst, w=w, directed=True), stable=False)
csr = CsrGraph(n=n, offsets=c.offsets.cpu().numpy(), targets=c.targets.cpu().numpy(),
               weights=c.weights.cpu().numpy(), directed=True)
del c, src, dst, w
torch.cuda.empty_cache()
yl = LabelVector(labels=y.cpu().numpy(), k=k)
p = prepare(csr, k, residency="device")
h_z = np.empty((n, k), dtype=np.float32)
embed_parallel(p, yl, out=h_z)
t0 = time.perf_counter()
embed_parallel(p, yl, out=h_z)
call = time.perf_counter() - t0
pipe = p._pipe_res
i = len(pipe.views) - 1
lo, hi, _, _ = pipe.views[i].span
h = i % pipe.HOST_SLOTS
out = {"call_s": call, "chunks": len(pipe.views)}
for threads in (16, 8, 4):
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        rc = io_lib().gee_io_expand_rows(_lib.ptr(pipe.hm[h]), _lib.ptr(pipe.hv[h]), _lib.ptr(pipe.hb[h]), hi - lo,
                                         k, ctypes.c_void_p(h_z.ctypes.data + lo * k * 4), threads)
        ts.append(time.perf_counter() - t0)
    out[f"expand_chunk_s_t{threads}"] = min(ts)
    out[f"expand_GBps_t{threads}"] = (hi - lo) * k * 4 / min(ts) / 1e9
t0 = time.perf_counter()
h_z.fill(0.0)
out["numpy_fill_GBps"] = h_z.nbytes / (time.perf_counter() - t0) / 1e9
print(json.dumps(out))
