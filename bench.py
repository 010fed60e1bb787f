#!/usr/bin/env python
"""Benchmark: MosaicBERT-Base seq-128 data-parallel training step on B200 (BASELINE.json metric
"non-pad tokens/sec & MFU").

One step = one optimizer step of the whole hot path on every rank: unpad index + MLM select (A1),
embedding (A3), 12 encoder layers forward (A4-A9), MLM head + CE forward/backward (A11), 12 layers
backward (A10, A4-A9 bwd), embedding backward, NCCL gradient allreduce overlapped with the backward
(A12), fused AdamW (F1).  The global batch is 4096 sequences at every N: each
rank runs accumulation = 4096 / (N x micro) micro-batches of 512 sequences x 128 per
optimizer step (8/N at C2), the gradient allreduce overlapping the last micro-step's backward.
Per-GPU work per micro-step is the same at every N: weak scaling.  (--accum 1: one micro-batch per
optimizer step, global batch 512 N.)

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--accum A] [--impl ours|reference]

Prints ONE JSON line on rank 0.  `--impl reference` times the fp64 CPU oracle (the reference arm of
this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

PEAK_DATASHEET = 2.25e15  # dense bf16 B200 (R23)
MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "non-pad tokens/sec & MFU, MosaicBERT-Base seq128 train step, 1/2/4/8 B200"
PAPER_TOKS = 1.1e6  # 8xA100-80GB, Table H1


def peaks():
    try:
        d = json.load(open(MEASURED))
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def workload_name(cfg):
    c = synth.CONFIGS[cfg]
    d = c.dims
    return (f"{cfg}: MosaicBERT-{'Large' if d.hidden == 1024 else 'Base'} {d.layers}L H{d.hidden} "
            f"heads{d.heads} GeGLU{d.intermediate} V{d.vocab} seq{c.seq_len} micro{c.micro_batch}/GPU "
            f"lengths={c.lengths} 30% MLM")


# --------------------------------------------------------------------------------------- clocks
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append((float(f[1]), float(f[2]), float(f[3]), f[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[3]) if v.lower() == "active"})
        loaded = [r for r in rows if r[2] > 300] or rows
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "power_w_median": statistics.median(r[2] for r in loaded), "samples": len(rows),
                "reasons": reasons}


# --------------------------------------------------------------------------------------- oracle arm
_PARAMS = {}


def oracle_sample(cfg: str, n_seq: int, seed: int = 0):
    """Bounded sample of the workload for the CPU oracle: the first n_seq sequences of the rank-0
    micro-batch with the full-depth model (same params as the GPU arm)."""
    c = synth.CONFIGS[cfg]
    batch = synth.make_batch(cfg, 1000 * int(cfg[1]) + 0)
    batch = {k: v[:n_seq] for k, v in batch.items()}
    if (cfg, seed) not in _PARAMS:
        _PARAMS[(cfg, seed)] = synth.make_model_params(c.dims, seed, "bert")
    return batch, _PARAMS[(cfg, seed)]


def time_oracle(cfg: str, n_seq: int, reps: int = 1):
    import oracle as O
    c = synth.CONFIGS[cfg]
    batch, params = oracle_sample(cfg, n_seq)
    params64 = {k: (v.astype(np.float64) if k != "layers" else
                    [{kk: vv.astype(np.float64) for kk, vv in l.items()} for l in v]) for k, v in params.items()}
    slopes = O.alibi_slopes(c.dims.heads)
    ntok = int(batch["attention_mask"].sum())
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.model_forward_backward(batch, params64, slopes, c.dims.ln_eps)
        ts.append(time.perf_counter() - t0)
    return ntok, ts


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_baseline(cfg: str, n_seq: int):
    """the oracle as it stands, 1 warm-up + 3 timed runs, median, on the host cores."""
    time_oracle(cfg, n_seq, reps=1)
    ntok, ts = time_oracle(cfg, n_seq, reps=3)
    med = statistics.median(ts)
    return {"value": ntok / med, "unit": "tokens/s", "cores": cpu_cores(), "cpu_model": cpu_model(), "kind": "oracle",
            "sample": f"first {n_seq} sequences of the rank-0 {cfg} micro-batch ({ntok} non-pad tokens), full-depth "
                      f"fp64 step (embedding, {synth.CONFIGS[cfg].dims.layers} layers fwd+bwd, head+CE); 1 warm-up "
                      f"+ median of 3 runs ({', '.join(f'{t:.1f}' for t in ts)} s)",
            "note": "unoptimised fp64 correctness oracle (numpy/OpenBLAS on the host cores), not a tuned baseline"}


def step_flops(cfg: str, lens, n_masked: int):
    """Algorithmic FLOPs of one micro-step: encoder GEMMs 6 (3H^2 + H^2 + 2IH + IH) per
    token and layer, attention 12 H l_b per token of a length-l_b sequence and layer (QK^T, PV forward
    + 4 backward products), MLM head 6 (H^2 + H V) per masked token.  (MFU instead credits 6 N per
    token, Eq. 3.)"""
    d = synth.CONFIGS[cfg].dims
    H, I, V, nl = d.hidden, d.intermediate, d.vocab, d.layers
    T = float(np.sum(lens))
    gemm = 6.0 * nl * (3 * H * H + H * H + 2 * I * H + I * H) * T
    attn = 12.0 * nl * H * float(np.sum(np.asarray(lens, dtype=np.float64) ** 2))
    head = 6.0 * (H * H + H * V) * n_masked
    return gemm + attn + head


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n_seq = min(args.oracle_seqs, 8)  # keeps the whole reference run within a few minutes
    ntok, _ = time_oracle(args.config, n_seq, reps=1) if args.warmup > 0 else (0, [])
    for _ in range(max(args.warmup - 1, 0)):
        time_oracle(args.config, n_seq, reps=1)
    ntok, ts = time_oracle(args.config, n_seq, reps=args.steps)
    total = sum(ts)
    val = ntok * len(ts) / total
    cores = cpu_cores()
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(ts), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config), "sample": f"first {n_seq} sequences of the rank-0 "
                   f"micro-batch ({ntok} non-pad tokens), full-depth model", "parallelism": "host cores"},
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cores, "cpu_model": cpu_model(), "kind": "oracle",
                         "sample": f"{n_seq} sequences x {synth.CONFIGS[args.config].seq_len}, {ntok} tokens"},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--oracle-seqs", type=int, default=8)
    ap.add_argument("--accum", type=int, default=None,
                    help="micro-steps per optimizer step (default: global batch 4096 sequences, P:177)")
    ap.add_argument("--nccl-sm-carveout", type=int, default=0,
                    help="leave this many SMs out of the persistent kernels' grids (NCCL kernels run there)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-balance", action="store_true",
                    help="N > 1: contiguous slices of the global batch instead of the LPT partition")
    ap.add_argument("--micro", type=int, default=None, help="override the per-GPU micro-batch")
    ap.add_argument("--dropout", type=float, default=0.0,
                    help="F2 feed-forward dropout p (P:152 trains with 0.1; the §8(a) hot path is p = 0, R13)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.nccl_sm_carveout:
        os.environ["MB_SM_CARVEOUT"] = str(args.nccl_sm_carveout)  # read by the library at first launch

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("MB_DIST_BACKEND", "nccl")  # "gloo": functional test of the N > 1 path only
    if backend != "nccl":
        local %= torch.cuda.device_count()  # (ranks may share a GPU; gloo kernels never wait on each other)
    torch.cuda.set_device(local)
    if world > 1 and backend == "nccl":
        # NCCL on a high-priority stream: when a persistent kernel's CTAs retire, the block scheduler
        # hands the freed SMs to a pending bucket allreduce before the next compute kernel
        opts = dist.ProcessGroupNCCL.Options()
        opts.is_high_priority_stream = True
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), pg_options=opts)
    elif world > 1:
        dist.init_process_group(backend)
    from paper_2312_17482_b200 import _lib as L
    from paper_2312_17482_b200.model import ModelDims, MosaicBert, param_count

    cfg = synth.CONFIGS[args.config]
    d = cfg.dims
    micro = args.micro or cfg.micro_batch
    dims = ModelDims(d.hidden, d.heads, d.intermediate, d.vocab, d.layers, d.ln_eps)
    params = synth.make_model_params(d, 0, "bert")  # random BERT init (never zeros: B200 is power-capped)
    model = MosaicBert(dims, params, device=f"cuda:{local}", process_group=None, dropout=args.dropout, seed=rank)
    del params
    n_params = param_count(dims)

    accum = args.accum or max(1, 4096 // (world * micro))  # global batch 4096

    # synthetic micro-batches for this rank (inputs resident in HBM for the device-timed value).
    # N > 1: every rank draws the same global batch (world x accumulation x micro sequences) and
    # takes its share of an LPT partition on the sequence lengths (per-rank nnz equal
    # to < 0.5 % on ragged batches, so no rank straggles); --no-balance: contiguous slices.
    nb = max(2, accum)
    host = []
    balance = None
    if world > 1:
        from paper_2312_17482_b200.balance import imbalance, lpt_partition
        per_rank = accum * micro
        imb = []
        for gi in range((nb + accum - 1) // accum):
            gb = synth.make_batch(cfg, 1000 * int(args.config[1]) + 7919 * gi, B=world * per_rank)
            lens_g = gb["attention_mask"].sum(1)
            parts = (lpt_partition(lens_g, world) if not args.no_balance else
                     [np.arange(r * per_rank, (r + 1) * per_rank) for r in range(world)])
            imb.append(imbalance(lens_g, parts))
            mine = parts[rank]
            for j in range(accum):
                sel = mine[j * micro:(j + 1) * micro]
                host.append({k: torch.from_numpy(np.ascontiguousarray(gb[k][sel])).pin_memory()
                             for k in ("input_ids", "attention_mask", "labels")})
        host = host[:nb]
        balance = {"method": "contiguous" if args.no_balance else "LPT on sequence length",
                   "max_rank_nnz_over_mean": 1.0 + max(imb)}
    else:
        for i in range(nb):
            b = synth.make_batch(cfg, 1000 * int(args.config[1]) + 17 * rank + i, B=micro)
            host.append({k: torch.from_numpy(b[k]).pin_memory() for k in ("input_ids", "attention_mask", "labels")})
    dev = [{k: v.cuda() for k, v in h.items()} for h in host]
    tokens = [int(h["attention_mask"].sum()) for h in host]
    lens = [h["attention_mask"].sum(1).numpy() for h in host]

    # (nnz, max_seqlen, n_masked) of each batch from its host copy: the step then needs no device->host
    # read of the unpad results (they are still computed on the device and verified one step later)
    metas = [MosaicBert.batch_meta(h["attention_mask"], h["labels"]) for h in host]
    flops = [step_flops(args.config, lens[i], metas[i][2]) for i in range(nb)]

    def micro_ids(i):
        return [(i * accum + j) % nb for j in range(accum)]

    def step(i, hostcopy=False, use_meta=True):
        mbs = []
        for j in micro_ids(i):
            b = dev[j]
            if hostcopy:
                for k in b:
                    b[k].copy_(host[j][k], non_blocking=True)
            mbs.append((b["input_ids"], b["attention_mask"], b["labels"]))
        return model.train_step(mbs, host_meta=[metas[j] for j in micro_ids(i)] if use_meta else None)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        return float(t.item())

    for i in range(args.warmup):
        step(i)
    barrier()

    # ---- device-timed value: inputs resident, K steps between CUDA events, max over ranks
    probe = L.Probe(1, capacity=2 * d.layers * accum * args.steps + 8)
    n0 = L.launch_count()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    profile_range = os.environ.get("MB_PROFILE_RANGE") == "1"  # nsys --capture-range=cudaProfilerApi
    with Clocks(local) as clk, probe:
        barrier()
        if profile_range:
            torch.cuda.profiler.start()
        evs[0].record()
        loss = None
        for i in range(args.steps):
            loss = step(i)
            evs[i + 1].record()
        barrier()
        if profile_range:
            torch.cuda.profiler.stop()
    model.check_meta()
    launches = (L.launch_count() - n0) // args.steps
    ms = evs[0].elapsed_time(evs[-1])
    per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    ms_max = max_over_ranks(ms)
    tok_step = sum_over_ranks(float(np.mean([sum(tokens[j] for j in micro_ids(i)) for i in range(args.steps)])))
    flop_step = sum_over_ranks(float(np.mean([sum(flops[j] for j in micro_ids(i)) for i in range(args.steps)])))
    value = tok_step * args.steps / (ms_max / 1e3)
    clocks = clk.summary()
    loss_val = sum_over_ranks(float(loss.item()))  # each rank holds its share of the global mean (R18)

    # ---- roofline of the dominant kernel (GeGLU up-projection GEMM, A8), timed inside the steps
    pk, src = peaks()
    gemm_ms = probe.times_ms()
    T = tokens[0]
    flops_gemm = 2.0 * T * d.hidden * 2 * d.intermediate  # algorithmic: T x H x 2I MACs per launch
    achieved = flops_gemm / (np.mean(gemm_ms) / 1e3) / 1e12 if gemm_ms else None
    peak_tf = pk.get("bf16_tflops_sustained") or pk.get("bf16_tflops")
    traffic = None
    tp = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("geglu_fwd_gemm_dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"kernel": "gemm_kernel PAIRED (A8 GeGLU up-projection: 2-CTA tcgen05 GEMM, paired W1|V tile, fused "
                          "bias + GeLU-gate epilogue)",
                "bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": (achieved / peak_tf) if achieved else None, "traffic": traffic,
                "peak_source": f"{src} bf16_tflops_sustained (kernel timed inside a long step)",
                "launches_timed": len(gemm_ms),
                "algorithmic_flops_per_launch": flops_gemm,
                "share_of_step": (sum(gemm_ms) / ms) if gemm_ms else None}

    # ---- e2e through the public API with host buffers (H2D of ids/mask/labels + D2H of the loss)
    e2e = None
    if not args.no_e2e:
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.steps):
            l_ = step(i, hostcopy=True)
            float(l_.item())
        e1.record()
        barrier()
        model.check_meta()
        ems = max_over_ranks(e0.elapsed_time(e1))
        # the same, for a loader that does not know (nnz, max_seqlen, n_masked) on the host: every
        # micro-step then reads the device index results back (one 16-byte D2H sync per micro-step)
        barrier()
        e0.record()
        for i in range(args.steps):
            l_ = step(i, hostcopy=True, use_meta=False)
            float(l_.item())
        e1.record()
        barrier()
        ems_sync = max_over_ranks(e0.elapsed_time(e1))
        h2d = accum * sum(int(v.numel() * v.element_size()) for v in host[0].values())
        e2e = {"value": tok_step * args.steps / (ems / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 4, "ms_per_step": ems / args.steps,
               "host_meta": "batch (nnz, max_seqlen, n_masked) from the host copy of each micro-batch (the "
                            "device index results are still computed and checked one micro-step later)",
               "without_host_meta": {"value": tok_step * args.steps / (ems_sync / 1e3), "unit": "tokens/s",
                                     "ms_per_step": ems_sync / args.steps,
                                     "d2h_bytes_per_step": 4 + 16 * accum}}

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_baseline(args.config, args.oracle_seqs)

    if rank == 0:
        tok_s = value
        mfu_ds = 6.0 * n_params * tok_s / (world * PEAK_DATASHEET)
        mfu_meas = 6.0 * n_params * tok_s / (world * pk["bf16_tflops"] * 1e12)
        flop_s = flop_step * args.steps / (ms_max / 1e3)
        q = np.quantile(per_step, [0.1, 0.5, 0.9])
        line = {
            "metric": METRIC, "value": tok_s, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None,  # BASELINE.md has no number for this metric on B200 (the paper's 8xA100 row is context)
            "step_ms_p10_p50_p90": [float(x) for x in q],
            "dtype": "bf16", "data": "synthetic (seeded; random BERT-init weights)",
            "config": {"workload": workload_name(args.config), "global_batch": micro * world * accum,
                       "micro_batch_per_gpu": micro, "accumulation": accum, "seq_len": cfg.seq_len,
                       "parallelism": f"dp{world}", "nccl_sm_carveout": args.nccl_sm_carveout,
                       "shard_balance": balance,
                       "non_pad_tokens_per_step": tok_step, "l2": "working set >> L2 (weights 275 MB + "
                       "activations ~25 GB per step), no flush needed",
                       "optimizer": "fused AdamW inside the step", "ffn_dropout": args.dropout},
            "mfu": {"datasheet_2.25PF": mfu_ds, "measured_peak": mfu_meas, "n_params": n_params,
                    "formula": "6 N tok/s / (G peak) (Eq. 3, P:608)"},
            "hfu": {"datasheet_2.25PF": flop_s / (world * PEAK_DATASHEET),
                    "measured_peak": flop_s / (world * pk["bf16_tflops"] * 1e12),
                    "measured_sustained": flop_s / (world * pk["bf16_tflops_sustained"] * 1e12),
                    "algorithmic_tflop_per_step": flop_step / 1e12,
                    "formula": "SURVEY 8(d) algorithmic FLOPs (GEMMs + attention at each sequence's own l + head on "
                               "the masked rows) / time / (G peak)"},
            "loss": loss_val,
            "clocks": clocks,
            "gpu_launches": int(launches),
            "roofline": roofline,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
