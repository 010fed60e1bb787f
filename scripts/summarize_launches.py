"""Summarise an ncu launch list CSV (gpu__time_duration.sum) of bench steps: per-kernel totals and
shares for the LAST step (launches after the last unpad_index_kernel)."""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
    rows.append((r["Kernel Name"], v * scale))
# last step = from the last unpad_index_kernel
starts = [i for i, (k, _) in enumerate(rows) if "unpad_index" in k or "unpad_count" in k]
step = rows[starts[-1]:] if starts else rows
tot = sum(t for _, t in step)
agg = defaultdict(lambda: [0, 0.0])
for k, t in step:
    name = re.sub(r"\(.*", "", k)
    name = re.sub(r"^void ", "", name)
    agg[name][0] += 1
    agg[name][1] += t
print(f"launches in last step: {len(step)}, serialized device time {tot/1e3:.2f} ms")
for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t/1e3:9.3f} ms {100*t/tot:6.2f}%  x{n:4d}  {name}")
if len(sys.argv) > 2:  # optional: per-launch times (us) of kernels matching a regex, in launch order
    rx = re.compile(sys.argv[2])
    print(" ".join(f"{t:.0f}" for k, t in step if rx.search(k)))
