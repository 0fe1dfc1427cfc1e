"""Dev tool: span-length statistics of the heavy rows per slot tile (C4): how
many arcs of the upper (sparse) tiles sit in spans long enough to be worth
the tile path?"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2402_04403_b200 import _lib, synth  # noqa: E402
from paper_2402_04403_b200._lib import check, lib, ptr  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph  # noqa: E402

src, dst, w, y, n, k, directed = synth.make_config(4)
g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
del src, dst, w
g.prepare_hot(k)
ts, T = 196608, 86
H = g.n_heavy
sentinel = g.n_hot + g.n_nodes
thr = torch.tensor([s * ts for s in range(T)] + [min(T * ts, sentinel), sentinel], dtype=torch.int64, device=g.device)
bounds = torch.empty((T + 2) * H, dtype=torch.int64, device=g.device)
check(lib.gee_tile_bounds(ptr(g.offsets), ptr(g.heavy_rows), H, ptr(g.targets), ptr(thr), T + 2, ptr(bounds),
                          _lib.stream_handle()), "b")
seg = (bounds.view(T + 2, H)[1:] - bounds.view(T + 2, H)[:-1])  # (T+1, H)
out = {"heavy_rows": H, "per_tile_range": {}}
for lo, hi in ((0, 21), (21, 42), (42, 86), (86, 87)):
    s = seg[lo:hi]
    tot = int(s.sum())
    row = {"arcs": tot, "spans": int((s > 0).sum())}
    for m in (8, 16, 32, 64, 128):
        sel = s >= m
        row[f"arcs_in_spans_ge_{m}"] = int(s[sel].sum())
        row[f"spans_ge_{m}"] = int(sel.sum())
    out["per_tile_range"][f"{lo}-{hi}"] = row
print(json.dumps(out, indent=1))
