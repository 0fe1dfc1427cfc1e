"""Resident host-result call on C4 vs the share of chunks copied out dense
(dev tool): prepare(residency='device') + embed_parallel(..., out=host)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2402_04403_b200 import CsrGraph, EdgeList, LabelVector, build_csr, embed_parallel, prepare, synth  # noqa
from paper_2402_04403_b200.stream import HostPipeline  # noqa: E402

src, dst, w, y, n, k, directed = synth.make_config(4)
c = build_csr(EdgeList(n=n, src=src, dst=dst, w=w, directed=True), stable=False)
csr = CsrGraph(n=n, offsets=c.offsets.cpu().numpy(), targets=c.targets.cpu().numpy(),
               weights=c.weights.cpu().numpy(), directed=True)
del c, src, dst, w
torch.cuda.empty_cache()
yl = LabelVector(labels=y.cpu().numpy(), k=k)
mode = sys.argv[1] if len(sys.argv) > 1 else "device"
p = prepare(csr, k, residency=mode)
h_z = np.empty((n, k), dtype=np.float32)
out = {}
for de in (0, 12, 8, 6, 4, 0, 8, 6):
    HostPipeline.DENSE_EVERY_RESIDENT = HostPipeline.DENSE_EVERY_STREAMED = de
    embed_parallel(p, yl, out=h_z)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        embed_parallel(p, yl, out=h_z)
        ts.append(time.perf_counter() - t0)
    out.setdefault(str(de), []).append(round(float(np.median(ts)) * 1e3, 1))
print(json.dumps(out))
