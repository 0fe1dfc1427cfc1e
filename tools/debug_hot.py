import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle
from paper_2402_04403_b200 import synth
from paper_2402_04403_b200.device import DeviceGraph, Embedder
scale, s, k = 19, 4_000_000, int(sys.argv[1]) if len(sys.argv) > 1 else 5
src, dst, w = synth.rmat_edges(scale, s, seed=11, weighted=False)
n = 1 << scale
y = synth.uniform_labels(n, k, seed=12)
exp = oracle.serial_embed(src.cpu().numpy(), dst.cpu().numpy(), None, y.cpu().numpy(), n, k)
for enable in (False, True):
    g = DeviceGraph.from_edges(src, dst, None, n, pull=True)
    g.prepare_hot(k, enable=enable)
    emb = Embedder(n, k)
    z = emb.embed(g, y, variant="pull").cpu().numpy()
    bad = np.argwhere(np.abs(z - exp) > 1e-4 * np.abs(exp) + 1e-12)
    print("enable", enable, "n_hot", g.n_hot, "bad entries", len(bad))
    if len(bad):
        rows = np.unique(bad[:, 0])
        print(" bad rows", rows[:20], len(rows))
        off = g.offsets.cpu().numpy()
        tr = (g.ensure_tile_plan() or g.tile_row).cpu().numpy()
        for r in rows[:5]:
            print("  row", r, "deg", off[r+1]-off[r], "start", off[r], "tile", off[r] // 4096, "z", z[r], "exp", exp[r])
        print(" tile_row around:", [(j, tr[j]) for j in range(len(tr)) if tr[j] in rows[:5] or (j+1 < len(tr) and tr[j] <= rows[0] < tr[j+1])][:5])
