"""Duplicate arcs in the prepared C4 pull layout (rows sorted by slot):
how many lookups / shared adds a duplicate-merging preparation would save,
by row class (dev tool)."""
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
t, off = g.targets, g.offsets
arcs = t.numel()
sentinel = g.n_hot + g.n_nodes
deg = off[1:] - off[:-1]
heavy_row = deg > g.HEAVY_ARCS
row_of = torch.repeat_interleave(torch.arange(g.n, device=t.device), deg)
dup = torch.zeros(arcs, dtype=torch.bool, device=t.device)
dup[1:] = (t[1:] == t[:-1]) & (row_of[1:] == row_of[:-1]) & (t[1:] != sentinel)
real = t != sentinel
hv = heavy_row[row_of]
print("arcs (padded)", arcs, "real", int(real.sum()))
print("duplicate arcs", int(dup.sum()), f"{dup.sum().item() / real.sum().item() * 100:.2f}% of real arcs")
print("  in heavy rows", int((dup & hv).sum()), f"{(dup & hv).sum().item() / (real & hv).sum().item() * 100:.2f}% of heavy arcs")
print("  in light rows", int((dup & ~hv).sum()), f"{(dup & ~hv).sum().item() / (real & ~hv).sum().item() * 100:.2f}% of light arcs")
