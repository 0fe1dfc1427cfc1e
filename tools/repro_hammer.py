"""Debug: hammer graph (two heavy rows) through the padded pull, phase by phase."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_04403_b200._lib import check, lib, ptr  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph, Embedder, _stream  # noqa: E402

s = 5000
dev = torch.device("cuda")
g = DeviceGraph.from_edges(torch.zeros(s, dtype=torch.int32), torch.ones(s, dtype=torch.int32),
                           torch.full((s,), 0.5), 2, device=dev)
g.prepare_hot(1)
print("padded", g.padded, "arcs", g.arcs, "offsets", g.offsets.tolist(), "targets uniq", g.targets.unique().tolist(),
      "w uniq", g.weights.unique().tolist(), "scale", g.scale_exp, "items", g.n_items, g.item_slot.tolist())
emb = Embedder(2, 1, dev)
y = torch.tensor([0, 1], dtype=torch.int32, device=dev)
emb.project(y, g=g)
print("table", emb.table[:8].tolist(), "counts", emb.counts.tolist(), "inv", emb.inv64.tolist())
emb.cls = torch.full((g.arcs + 64,), 7, dtype=torch.uint8, device=dev)
check(lib.gee_gather_labels(ptr(g.targets), g.arcs, ptr(emb.table), g.n_hot, 1, ptr(emb.cls), _stream()), "g")
print("cls uniq", emb.cls[:g.arcs].unique().tolist())
z = torch.full((2, 1), -1.0, device=dev)
check(lib.gee_reduce_blocks_pad8(ptr(g.offsets), g.n, ptr(emb.cls), ptr(g.weights), g.scale_exp, ptr(emb.inv64), 1,
                                 g.HEAVY_ARCS, ptr(z), _stream()), "b")
torch.cuda.synchronize()
print("after blocks", z.tolist())
check(lib.gee_reduce_heavy(ptr(emb.cls), ptr(g.weights), g.arcs, g.scale_exp, ptr(emb.inv64), 1, ptr(g.item_first),
                           ptr(g.item_end), ptr(g.item_row), ptr(g.item_slot), g.n_items, ptr(g.mega_rows), g.n_mega,
                           None, ptr(emb.counter), ptr(z), _stream()), "h")
torch.cuda.synchronize()
print("after heavy", z.tolist())
