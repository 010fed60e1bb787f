"""Aggregate an ncu counters CSV (scripts/profile_counters.sh) over the LAST bench step: per kernel,
launches, mean duration, achieved DRAM GB/s, tensor-pipe / DRAM / SM utilisation (% of peak)."""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(lines))
launch = defaultdict(dict)
order = []
for r in rows:
    key = (r["ID"], r["Kernel Name"])
    if key not in launch:
        order.append(key)
    v = float(r["Metric Value"].replace(",", "")) if r["Metric Value"] else 0.0
    unit = r.get("Metric Unit", "")
    name = r["Metric Name"]
    if name == "gpu__time_duration.sum":
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
    elif name.startswith("dram__bytes"):
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    launch[key][name] = v
starts = [i for i, (_, k) in enumerate(order) if "unpad_index" in k or "unpad_count" in k]
step = order[starts[-1]:] if starts else order
agg = defaultdict(lambda: defaultdict(float))
for key in step:
    m = launch[key]
    nm = re.sub(r"\(.*", "", key[1]).replace("void ", "").replace("mb::<unnamed>::", "")
    a = agg[nm]
    a["n"] += 1
    for k, v in m.items():
        a[k] += v
tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
print(f"| kernel | launches | mean us | share | DRAM GB/s | tensor pipe % | DRAM % | SM % |")
print("|---|---|---|---|---|---|---|---|")
for nm, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    n = a["n"]
    t = a["gpu__time_duration.sum"]
    gbs = (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / (t * 1e-6) / 1e9 if t else 0
    print(f"| `{nm}` | {int(n)} | {t / n:.1f} | {100 * t / tot:.1f} % | {gbs:.0f} | "
          f"{a['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'] / n:.1f} | "
          f"{a['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'] / n:.1f} | "
          f"{a['sm__throughput.avg.pct_of_peak_sustained_elapsed'] / n:.1f} |")
