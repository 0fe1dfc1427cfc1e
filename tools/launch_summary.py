"""Summarise an ncu launch list (gpu__time_duration.sum per launch) of a
bench run: per kernel launches, mean / total time (dev + profiles tool)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
per = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    per.setdefault(name, []).append(float(r[vi].replace(",", "")) * scale[r[ui]])
ours = ("k_label_hist", "k_inv", "k_gather", "k_reduce_blocks", "k_reduce_heavy", "k_heavy_finalize")  # k_gather: packed, scatter, tiles
steps = int(sys.argv[2]) if len(sys.argv) > 2 else None
print(f"{'kernel':48s} {'launches':>8s} {'mean ms':>10s} {'total ms':>10s}")
step_total = 0.0
for name, t in per.items():
    print(f"{name[:48]:48s} {len(t):8d} {sum(t) / len(t):10.4f} {sum(t):10.3f}")
if steps:
    print("\nper-step share of the pull path (last", steps, "launches of each path kernel):")
    last = {n: t[-steps:] for n, t in per.items() if n.startswith(ours)}
    tot = sum(sum(t) / len(t) for t in last.values())
    for n, t in last.items():
        m = sum(t) / len(t)
        print(f"  {n[:46]:46s} {m:9.4f} ms  {100 * m / tot:5.1f}%")
    print(f"  {'sum (serialised, cold-cache ncu timing)':46s} {tot:9.4f} ms")
