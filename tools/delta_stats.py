"""Compressibility of the prepared C4 targets (rows sorted by slot, padded to 8):
bytes per arc for per-8-arc-group byte-width delta coding (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_04403_b200 import synth  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph  # noqa: E402

src, dst, w, y, n, k, _ = synth.make_config(4)
g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
del src, dst, w
torch.cuda.empty_cache()
g.prepare_hot(k)
t = g.targets
off = g.offsets
arcs = t.numel()
print("arcs", arcs, "n_hot", g.n_hot)
hist = torch.zeros(5, dtype=torch.int64, device=t.device)
step = 1 << 28
# row start flags for group boundaries
starts = torch.zeros(arcs + 1, dtype=torch.bool, device=t.device)
starts[off[:-1].clamp(max=arcs)] = True
for a in range(0, arcs, step):
    b = min(arcs, a + step)
    x = t[a:b].long()
    prev = torch.empty_like(x)
    prev[1:] = x[:-1]
    prev[0] = t[a - 1].long() if a else 0
    d = x - prev
    d = torch.where(starts[a:b], x, d)  # row's first arc: absolute slot
    assert bool((d >= 0).all())
    nb = torch.where(d < (1 << 8), 1, torch.where(d < (1 << 16), 2, torch.where(d < (1 << 24), 3, 4)))
    gw = nb.view(-1, 8).amax(1)
    hist += torch.bincount(gw, minlength=5)[:5]
tot = int(hist.sum())
bpa = float((hist * torch.arange(5, device=t.device)).sum()) * 8 / arcs + 0.25
print("groups by width", hist.tolist(), "bytes/arc (+2-bit ctl)", round(bpa, 3), "vs 4")
