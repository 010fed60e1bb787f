"""Print the key ncu metrics of a .ncu-rep (first kernel): duration, throughput, DRAM bytes, tensor
pipe, occupancy, top warp-stall reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum", "launch__grid_size"]
for k in keys:
    if k in m:
        print(f"{k:70s} {m[k]} {u.get(k, '')}")
for k in sorted(m):
    if ("tensor" in k or "tmem" in k.lower() or "utc" in k.lower()) and "pct" in k and m[k] not in ("", "0"):
        print(f"{k:70s} {m[k]} {u.get(k, '')}")
stalls = [(k, m[k]) for k in m if k.startswith("smsp__average_warp_latency_issue_stalled") or
          k.startswith("smsp__pcsamp_warps_issue_stalled")]
st = []
for k, v in stalls:
    try:
        st.append((float(v.replace(",", "")), k))
    except ValueError:
        pass
for v, k in sorted(st, reverse=True)[:12]:
    print(f"  stall {k:80s} {v}")
