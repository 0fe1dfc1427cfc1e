"""Write profiles/ncu_traffic.json (dram bytes per launch per kernel) from
one `ncu --set full` capture of bench.py (bench.py's roofline.traffic)."""
import csv
import json
import subprocess
import sys

rep, workload, out = sys.argv[1], sys.argv[2], sys.argv[3]
metrics = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "lts__t_sector_hit_rate.pct"]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                     capture_output=True, text=True).stdout
r = list(csv.reader(txt.splitlines()))
h, units = r[0], r[1]
ki = h.index("Kernel Name")
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
        "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6, "%": 1.0}
kern = {}
for x in r[2:]:
    name = x[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "").split("<")[0]
    v = {m: float(x[h.index(m)].replace(",", "")) * mult[units[h.index(m)]] for m in metrics}
    kern[name] = {"dram_bytes_read": v["dram__bytes_read.sum"], "dram_bytes_write": v["dram__bytes_write.sum"],
                  "dram_bytes_per_launch": v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"],
                  "ncu_ms": v["gpu__time_duration.sum"], "l2_hit_pct": v["lts__t_sector_hit_rate.pct"]}
json.dump({"workload": workload, "source": rep.split("/")[-1], "kernels": kern}, open(out, "w"), indent=1)
print(json.dumps(kern, indent=1))
