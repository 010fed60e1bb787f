"""Top SASS instructions by warp-stall samples of an .ncu-rep (ncu --page source --print-source sass)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
recs = []
for i, r in enumerate(rows[2:]):
    try:
        recs.append((int(r[ist]), i, r[ia], r[isrc]))
    except (ValueError, IndexError):
        pass
tot = sum(x[0] for x in recs)
print(f"total samples {tot}")
for s, i, a, src in sorted(recs, reverse=True)[:n]:
    print(f"{s:6d} {100*s/tot:5.1f}%  #{i:5d} {a}  {src}")
