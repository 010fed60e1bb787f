"""Diagnostic: phase timeline of the long-forward softmax warpgroups and MMA issuer on CTA 0
(build with scripts/build_diag.sh trace "-DMB_TRACE_L2=1", run with MB_LIBRARY=ab/libmosaicbert_trace.so).
usage: l2_trace.py B L"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

os.environ.setdefault("MB_LIBRARY", "ab/libmosaicbert_trace.so")
import runpy  # noqa: E402

runpy.run_path(os.path.join(os.path.dirname(__file__), "attn_bench.py"), run_name="__main__")
from paper_2312_17482_b200 import _lib  # noqa: E402

buf = np.zeros(2 * 16 * 8 + 2 * 8 * 16, dtype=np.int64)
assert _lib.lib().mb_diag_l2_trace(buf.ctypes.data_as(C.c_void_p)) == 0
tr = buf[:256].reshape(2, 16, 8)
mt = buf[256:].reshape(2, 8, 16)
t0 = tr[0, 0, 0]
ev = ["waitS", "S_in", "S_ld", "scores", "pv_ok", "exps", "p_rdy"]
for t in range(2):
    print(f"warpgroup {t}: per tile, clocks relative to WG0 tile 0 start")
    for i in range(16):
        row = tr[t, i, :7] - t0
        print(f"  tile {i:2d} " + " ".join(f"{e}={v:7d}" for e, v in zip(ev, row)) +
              f"  | S: enter={mt[t, 2, i] - t0:7d} kv_ok={mt[t, 3, i] - t0:7d} iss={mt[t, 0, i] - t0:7d}"
              f"  PV: enter={mt[t, 4, i] - t0:7d} iss={mt[t, 1, i] - t0:7d} mmas_out={mt[t, 6, i] - t0:7d}")
for t in range(2):
    print(f"WG{t} issuer: S MMAs issue {np.mean(mt[t, 5] - mt[t, 0]):.0f} clk, PV MMAs issue {np.mean(mt[t, 6] - mt[t, 1]):.0f} clk")
for t in range(2):
    d = np.diff(tr[t, :, :7], axis=1)
    per = np.diff(tr[t, :, 0])
    print(f"WG{t} mean phase durations: " + " ".join(f"{ev[k]}->{ev[k + 1]} {d[:, k].mean():.0f}" for k in range(6)) +
          f" | tile period {per.mean():.0f}")
