"""Top SASS lines by warp-stall samples from `ncu --page source --csv` of a .ncu-rep."""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
rows.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
print(f"total samples {tot}")
for r in rows[:n]:
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{100*s/tot:5.1f}%  {r['Address'][-5:]}  {r['Source'].strip()[:90]}")
