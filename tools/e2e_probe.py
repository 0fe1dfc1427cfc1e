"""Where does the streamed e2e time go on C4? (dev tool)

Through prepare() + embed_parallel as bench.py does, then on the prepared
pipeline's own buffers:
  copy_in     every chunk's H2D (labels, hot tier, offsets, packed streams) alone;
  copy_both   the same with the row-sparse Z copy-out (last call's sizes) on
              the D2H stream at the same time;
  no_expand   the full call with the host expansion skipped (Z wrong; timing only);
  full        the full call.
Wall clock, median of 3."""
import json
import os
import sys
import time
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2402_04403_b200 import LabelVector, embed_parallel, prepare, synth  # noqa: E402


def med(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)) * 1e3


def main():
    chunks = int(os.environ.get("CHUNKS", "32"))
    src, dst, w, y, n, k, directed = synth.make_config(4)
    g = types.SimpleNamespace(src=src, dst=dst, w=w)
    del src, dst, w
    csr_h = bench.host_csr_from_coo(g, n, directed)
    y_h = LabelVector(labels=y.cpu().numpy(), k=k)
    prep = prepare(csr_h, k, chunks=chunks)
    h_z = np.empty((n, k), dtype=np.float32)
    embed_parallel(prep, y_h, out=h_z)
    pipe = prep._pipe
    out = {"chunks": chunks, "h2d_GB": prep.h2d_bytes_per_call / 1e9}
    out["full_ms"] = med(lambda: embed_parallel(prep, y_h, out=h_z))
    out["d2h_GB"] = pipe.d2h_bytes / 1e9
    h_y = prep._register(np.ascontiguousarray(y_h.labels, dtype=np.int32))

    def copy_in():
        with torch.cuda.stream(pipe.s_in):
            pipe.d_y.copy_(h_y, non_blocking=True)
            for d, h in zip(pipe.d_hot or [], pipe.h_hot or []):
                d.copy_(h, non_blocking=True)
            for i, v in enumerate(pipe.views):
                b = i & 1
                lo, hi, a0, a1 = v.span
                ho = pipe.h_off[i]
                (pipe.d_off32 if ho.dtype == torch.int32 else pipe.d_off)[b][:hi - lo + 1].copy_(ho, non_blocking=True)
                pipe.d_ctl[b][:pipe.h_ctl[i].numel()].copy_(pipe.h_ctl[i], non_blocking=True)
                pipe.d_pay[b][:pipe.h_pay[i].numel()].copy_(pipe.h_pay[i], non_blocking=True)
                if pipe.weighted:
                    if pipe.h_wctl[i].numel():
                        pipe.d_wctl[b][:pipe.h_wctl[i].numel()].copy_(pipe.h_wctl[i], non_blocking=True)
                    pipe.d_wpay[b][:pipe.h_wpay[i].numel()].copy_(pipe.h_wpay[i], non_blocking=True)
        pipe.s_in.synchronize()

    out["copy_in_ms"] = med(copy_in)
    out["copy_in_GBps"] = out["h2d_GB"] / out["copy_in_ms"] * 1e3
    pipe._sparse_slots()
    per = int(pipe.d2h_bytes) // max(1, len(pipe.views))
    dbuf = torch.empty(per // 4 + 1, dtype=torch.float32, device=pipe.device)
    hbuf = [pipe.hv[h][:per // 4 + 1] for h in range(pipe.HOST_SLOTS)]

    def copy_both():
        with torch.cuda.stream(pipe.s_out):
            for i in range(len(pipe.views)):
                hbuf[i % len(hbuf)].copy_(dbuf, non_blocking=True)
        copy_in()
        pipe.s_out.synchronize()

    out["copy_both_ms"] = med(copy_both)
    real_expand = pipe._expand
    pipe._expand = lambda i, e_out, hz: e_out[i].synchronize()
    out["no_expand_ms"] = med(lambda: embed_parallel(prep, y_h, out=h_z))
    pipe._expand = real_expand
    out["full_again_ms"] = med(lambda: embed_parallel(prep, y_h, out=h_z))
    out["expand_threads"] = {}
    for t in (5, 6, 7, 8, 9, 10, 12):
        pipe.EXPAND_THREADS = t
        out["expand_threads"][t] = med(lambda: embed_parallel(prep, y_h, out=h_z))
    pipe.EXPAND_THREADS = None
    prep_r = None
    prep.close()
    prep_r = prepare(csr_h, k, chunks=chunks, residency="device")
    embed_parallel(prep_r, y_h, out=h_z)
    out["resident_ms"] = med(lambda: embed_parallel(prep_r, y_h, out=h_z))
    pr = prep_r._pipe_res
    out["resident_expand_threads"] = {}
    for t in (12, 14, 15, 16):
        pr.EXPAND_THREADS = t
        out["resident_expand_threads"][t] = med(lambda: embed_parallel(prep_r, y_h, out=h_z))
    pr.EXPAND_THREADS = None
    import os as _os
    out["cpus"] = _os.cpu_count()
    out["affinity"] = len(_os.sched_getaffinity(0))
    print(json.dumps(out), flush=True)
    prep_r.close()


if __name__ == "__main__":
    main()
