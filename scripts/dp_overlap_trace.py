"""Data-parallel overlap trace (nsys is not in this image; CUPTI through torch.profiler instead).

Run under torchrun on N GPUs, e.g.
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \\
      --master-port 29511 scripts/dp_overlap_trace.py --config C2
Each rank times one optimizer step (SURVEY 8.0 accumulation, the bucket allreduces issued during
the last micro-step's backward) under the profiler, writes its chrome trace to
gpurun_out/dp_trace_rank<r>.json and prints one JSON line: NCCL kernel time, the part of it that
overlaps this library's kernels (mb::) on the same GPU, and the exposed remainder.  MB_SM_CARVEOUT=k leaves k SMs out of the persistent grids (room for NCCL CTAs);
NCCL_MAX_NCHANNELS / NCCL_NVLS_ENABLE are passed through to NCCL unchanged.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def intervals(events, pred):
    return sorted((e["ts"], e["ts"] + e["dur"]) for e in events if pred(e["name"]))


def overlap(a, b):
    """Total length of the intersection of two sorted interval lists."""
    tot, j = 0.0, 0
    for s, e in a:
        while j < len(b) and b[j][1] <= s:
            j += 1
        k = j
        while k < len(b) and b[k][0] < e:
            tot += max(0.0, min(e, b[k][1]) - max(s, b[k][0]))
            k += 1
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--accum", type=int, default=None)
    ap.add_argument("--force-dp", action="store_true",
                    help="one rank: still open an NCCL group and run the data-parallel path (bucket allreduces)")
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    backend = os.environ.get("MB_DIST_BACKEND", "nccl")
    if world > 1 or args.force_dp:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        if backend == "nccl":
            opts = dist.ProcessGroupNCCL.Options()
            opts.is_high_priority_stream = True
            dist.init_process_group("nccl", device_id=torch.device("cuda", local), pg_options=opts)
        else:
            dist.init_process_group(backend)
    from paper_2312_17482_b200.model import ModelDims, MosaicBert
    cfg = synth.CONFIGS[args.config]
    d = cfg.dims
    model = MosaicBert(ModelDims(d.hidden, d.heads, d.intermediate, d.vocab, d.layers, d.ln_eps),
                       synth.make_model_params(d, 0, "bert"), device=f"cuda:{local}", seed=rank)
    if args.force_dp:
        model._dp = lambda: True
    accum = args.accum or max(1, 4096 // (world * cfg.micro_batch))
    mbs, metas = [], []
    for i in range(accum):
        b = synth.make_batch(cfg, 5000 + 17 * rank + i, B=cfg.micro_batch)
        mbs.append(tuple(torch.from_numpy(b[k]).cuda() for k in ("input_ids", "attention_mask", "labels")))
        metas.append(MosaicBert.batch_meta(b["attention_mask"], b["labels"]))
    for _ in range(2):
        model.train_step(mbs, host_meta=metas)
    torch.cuda.synchronize()
    if world > 1 or args.force_dp:
        dist.barrier()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        model.train_step(mbs, host_meta=metas)
        torch.cuda.synchronize()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", f"dp_trace_rank{rank}.json")
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel" and "dur" in e]
    ours = intervals(ev, lambda n: "mb::" in n)
    nccl = intervals(ev, lambda n: "nccl" in n.lower())
    line = {"rank": rank, "world": world, "backend": backend, "config": args.config, "accumulation": accum,
            "sm_carveout": int(os.environ.get("MB_SM_CARVEOUT", "0")),
            "mb_kernel_us": sum(e - s for s, e in ours), "nccl_kernel_us": sum(e - s for s, e in nccl),
            "nccl_overlapped_us": overlap(nccl, ours),
            "nccl_exposed_us": sum(e - s for s, e in nccl) - overlap(nccl, ours),
            "trace": os.path.relpath(path, ROOT)}
    print(json.dumps(line), flush=True)
    if world > 1 or args.force_dp:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
