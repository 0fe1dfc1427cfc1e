"""Row-degree distribution of the C4 symmetric CSR (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_04403_b200 import synth  # noqa: E402
from paper_2402_04403_b200.device import DeviceGraph  # noqa: E402

src, dst, w, y, n, k, _ = synth.make_config(4)
g = DeviceGraph.from_edges(src, dst, w, n, pull=True)
d = (g.offsets[1:] - g.offsets[:-1])
arcs = float(d.sum())
nz = int((d > 0).sum())
print("rows", n, "nonempty", nz, "arcs", arcs)
for lo, hi in [(1, 1), (2, 8), (9, 16), (17, 32), (33, 64), (65, 256), (257, 2048), (2049, 1 << 40)]:
    m = (d >= lo) & (d <= hi)
    print(f"deg {lo:>5}-{hi:<12} rows {int(m.sum()):>11} ({m.sum().item() / nz * 100:5.1f}% of nonempty) "
          f"arcs {d[m].sum().item() / arcs * 100:5.1f}%")
