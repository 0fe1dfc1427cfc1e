"""Where do C4's label lookups go?  (diagnostic for the gather design)

For every arc of the prepared pull layout (padded, slot-sorted, hot-encoded):
light vs heavy row (> 2048 arcs), and the slot tier the lookup hits (pad
sentinel / shared-memory head / rest of the hot tier / cold).  For the
lookups that miss the head, the number of distinct 32-byte sectors per
32-arc warp instruction (the L2 requests the gather issues), for u8 labels
and for 6-bit labels packed 5 per word.  Also: for heavy rows, how many
distinct (row, hot tile) segments a tiled gather would write, for tiles of
T slots.
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2402_04403_b200 import synth  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else None
src, dst, w, y, n, k, directed = synth.make_config(4, scale_override=scale)
g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
del src, dst, w
torch.cuda.empty_cache()
g.prepare_hot(k)
tgt, off = g.targets, g.offsets
arcs = tgt.numel()
HEAD = 122880
sent = g.n_hot + g.n_nodes
deg = off[1:] - off[:-1]
heavy_row = deg > 2048
out = {"arcs_padded": arcs, "n_hot": g.n_hot, "heavy_rows": int(heavy_row.sum()),
       "heavy_arcs": int(deg[heavy_row].sum())}
cnt = torch.zeros(2, 4, dtype=torch.int64, device="cuda")
sect8 = torch.zeros(2, dtype=torch.int64, device="cuda")
sect6 = torch.zeros(2, dtype=torch.int64, device="cuda")
chunk = 1 << 28
TILES = (65536, 131072, 245760)
EDGES_R = [0, 122880, 245760, 491520, 1 << 20, 1 << 22, 1 << 24]
rank_hist = torch.zeros(2, len(EDGES_R) + 1, dtype=torch.int64, device="cuda")
bounds_r = torch.tensor(EDGES_R[1:], device="cuda")
segs = {T: 0 for T in TILES}
for a in range(0, arcs - arcs % 32, chunk):
    b = min(arcs - arcs % 32, a + chunk)
    t = tgt[a:b].long()
    e = torch.arange(a, b, device="cuda")
    row = torch.searchsorted(off, e, right=True) - 1
    hv = heavy_row[row].long()
    tier = torch.where(t == sent, 0, torch.where(t < HEAD, 1, torch.where(t < g.n_hot, 2, 3)))
    cnt.view(-1).index_add_(0, hv * 4 + tier, torch.ones_like(t))
    miss = tier >= 2
    bk = torch.where(tier == 0, torch.full_like(t, len(EDGES_R)), torch.bucketize(t, bounds_r, right=True))
    bk = torch.where((tier == 3), torch.full_like(t, len(EDGES_R) - 1), bk)
    rank_hist.view(-1).index_add_(0, hv * (len(EDGES_R) + 1) + bk, torch.ones_like(t))
    for table, div in ((sect8, 32), (sect6, 40)):
        s = torch.where(miss, t // div, torch.full_like(t, -1)).view(-1, 32)
        s, _ = torch.sort(s, dim=1)
        new = torch.ones_like(s, dtype=torch.bool)
        new[:, 1:] = s[:, 1:] != s[:, :-1]
        new &= s >= 0
        hvw = hv.view(-1, 32)[:, 0]
        table.index_add_(0, hvw, new.sum(1))
    rs = torch.zeros_like(hv, dtype=torch.bool)
    rs[1:] = row[1:] != row[:-1]
    rs[0] = True
    for T in TILES:
        tile = torch.where(t < g.n_hot, t // T, torch.full_like(t, -1))
        nw = torch.ones_like(rs)
        nw[1:] = (tile[1:] != tile[:-1])
        segs[T] += int((nw | rs)[(hv > 0) & (tile >= 0)].sum())
    del t, e, row, hv, tier, miss
names = ["pad", "head", "hot", "cold"]
for hv, lab in ((0, "light"), (1, "heavy")):
    out[lab] = {nm: int(cnt[hv, i]) for i, nm in enumerate(names)}
    out[lab]["l2_sectors_u8"] = int(sect8[hv])
    out[lab]["l2_sectors_6bit"] = int(sect6[hv])
for T in TILES:
    out[f"heavy_hot_segments_T{T}"] = segs[T]
labels_r = [f"<{b}" for b in EDGES_R[1:]] + ["cold", "pad"]
for hv, lab in ((0, "light"), (1, "heavy")):
    out[lab + "_by_rank"] = {labels_r[i]: int(rank_hist[hv, i]) for i in range(len(labels_r))}
print(json.dumps(out, indent=1))
