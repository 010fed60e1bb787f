"""Per-instruction warp-stall breakdown of an .ncu-rep (SASS view): the hottest instructions with
their top stall reasons, plus the per-reason totals.   usage: ncu_stalls.py rep [N] [lo hi]"""
import csv
import io
import subprocess
import sys

R = ["barrier", "branch_resolving", "dispatch_stall", "drain", "imc_miss", "lg_throttle", "long_scoreboard",
     "math_pipe_throttle", "membar", "mio_throttle", "misc", "no_instructions", "not_selected", "selected",
     "short_scoreboard", "sleeping", "tex_throttle", "wait"]
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 1 << 30)
mets = ",".join(f"smsp__pcsamp_warps_issue_stalled_{r}" for r in R)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--metrics", mets],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
cols = [(i, h.replace("stall_", "")) for i, h in enumerate(hdr) if h.startswith("stall_")]
recs = []
tot = {}
for k, r in enumerate(rows[2:]):
    if not (lo <= k < hi):
        continue
    vals = {nm: int(r[i] or 0) for i, nm in cols}
    for a, b in vals.items():
        tot[a] = tot.get(a, 0) + b
    recs.append((sum(vals.values()), k, r[1].strip(), vals))
T = sum(tot.values()) or 1
print("totals:", ", ".join(f"{a} {100*b/T:.1f}%" for a, b in sorted(tot.items(), key=lambda x: -x[1]) if b))
for s, k, src, vals in sorted(recs, reverse=True)[:n]:
    top = ", ".join(f"{a}:{b}" for a, b in sorted(vals.items(), key=lambda x: -x[1])[:3] if b)
    print(f"{s:6d} {100*s/T:5.1f}% #{k:5d} {src[:70]:70s} {top}")
