"""Dynamic instruction mix (warp-level instructions executed, by opcode) of a .ncu-rep's kernel,
from `ncu --page source --csv --print-source sass`."""
import csv, io, re, subprocess, sys
from collections import Counter
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
mix, stall = Counter(), Counter()
for r in rows:
    src = re.sub(r"^@!?U?P\w+\s+", "", r["Source"].strip())
    op = src.split(" ")[0].split(".")[0] if src else "?"
    mix[op] += int(r["Instructions Executed"] or 0)
    stall[op] += int(r["Warp Stall Sampling (All Samples)"] or 0)
tot, stot = sum(mix.values()), sum(stall.values())
print(f"warp instructions {tot}")
for op, n in mix.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{op:12s} {n:12d} {100*n/tot:5.1f}%   stall-samples {100*stall[op]/max(1,stot):5.1f}%")
