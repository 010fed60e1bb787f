"""Top SASS lines by warp-stall samples from `ncu --page source --csv` of a .ncu-rep, with each
line's two dominant stall reasons."""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
key = "Warp Stall Sampling (All Samples)"
tot = sum(int(r[key] or 0) for r in rows)
stall_cols = [k for k in rows[0] if k.startswith("stall_") and not k.endswith("_not_issued")]
rows.sort(key=lambda r: -int(r[key] or 0))
print(f"total samples {tot}")
for r in rows[:n]:
    s = int(r[key] or 0)
    rs = sorted(((float(r[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
    why = ",".join(f"{c}:{int(v)}" for v, c in rs if v > 0)
    print(f"{100*s/tot:5.1f}%  {r['Address'][-5:]}  {r['Source'].strip()[:70]:70s} {why}")
