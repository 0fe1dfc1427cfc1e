import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2402_04403_b200 import synth
from paper_2402_04403_b200.device import DeviceGraph
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
src, dst, w, y, n, k, directed = synth.make_config(4, scale_override=scale if scale != 27 else None)
g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
del src, dst, w
tr = (g.ensure_tile_plan() or g.tile_row).cpu().numpy().astype(np.int64)
off = g.offsets
rows = np.diff(tr)
deg = (off[1:] - off[:-1])
nonempty = int((deg > 0).sum())
print("n", n, "arcs", g.arcs, "tiles", len(rows), "nonempty rows", nonempty, "frac", nonempty / n)
print("rows/tile mean", rows.mean(), "p50", np.percentile(rows, 50), "p90", np.percentile(rows, 90), "p99", np.percentile(rows, 99), "max", rows.max())
win = np.ceil(np.maximum(rows, 1) / 256).astype(np.int64)
print("windows total", win.sum(), "tiles with >1 window", int((win > 1).sum()), "max windows", win.max())
# nonempty rows per tile
nz = torch.cumsum((deg > 0).to(torch.int64), 0).cpu().numpy()
nzc = np.concatenate([[0], nz])
nz_tile = nzc[tr[1:]] - nzc[tr[:-1]]
print("nonempty/tile mean", nz_tile.mean(), "p99", np.percentile(nz_tile, 99), "max", nz_tile.max())
