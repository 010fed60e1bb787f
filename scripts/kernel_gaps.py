"""Idle time between consecutive kernels of one bench step (CUPTI via torch.profiler): how much of
the device-timed step is launch gaps rather than kernel time.  Diagnostic only.
usage: python scripts/kernel_gaps.py [C2]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2312_17482_b200.model import ModelDims, MosaicBert  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
d = cfg.dims
model = MosaicBert(ModelDims(d.hidden, d.heads, d.intermediate, d.vocab, d.layers, d.ln_eps),
                   synth.make_model_params(d, 0, "bert"))
b = synth.make_batch(cfg, 2000, B=cfg.micro_batch)
dev = [torch.from_numpy(b[k]).cuda() for k in ("input_ids", "attention_mask", "labels")]
for _ in range(3):
    model.train_step([tuple(dev)])
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    model.train_step([tuple(dev)])
    torch.cuda.synchronize()
path = "/tmp/kernel_gaps_trace.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
start = np.array([e["ts"] for e in ev])
dur = np.array([e["dur"] for e in ev])
end = start + dur
gaps = start[1:] - end[:-1]
span = end[-1] - start[0]
print(f"kernels {len(ev)}  span {span / 1e3:.2f} ms  busy {dur.sum() / 1e3:.2f} ms  "
      f"gaps {gaps.clip(min=0).sum() / 1e3:.3f} ms ({100 * gaps.clip(min=0).sum() / span:.1f} %)")
print(f"gap us: median {np.median(gaps):.2f}  p90 {np.percentile(gaps, 90):.2f}  max {gaps.max():.1f}")
big = np.argsort(-gaps)[:8]
for i in big:
    print(f"  {gaps[i]:8.1f} us  after {ev[i]['name'][:60]}  before {ev[i + 1]['name'][:60]}")
