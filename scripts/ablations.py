"""F3 — the paper's throughput ablations re-measured on B200 with this repo's kernels.

  ln:      bf16 LayerNorm vs fp32-activation LayerNorm (same kernel designs), per C2 step
  glu:     fused GLU (paired-tile GEMM + GeGLU epilogues) vs naive GLU (two projection
           GEMMs + elementwise kernels saving the pre-activations), per C2 step
  unpad:   varlen (unpadded) train step vs the same batch run padded (every row treated as full
           length L), C5 batch (lognormal lengths, ~50 % padding), non-pad tokens/s
  vocab:   decoder vocabulary 30528 (multiple of 64) vs 30522, full C2 train step
  dropout: F2 feed-forward dropout 0.1 vs none, full C2 train step

Prints one JSON object (and writes it to the path given as argv[1], if any).  Times are CUDA-event
means over repeated launches on one GPU (B200, power-capped clocks as they come)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2312_17482_b200 import _lib as L  # noqa: E402
from paper_2312_17482_b200.model import ModelDims, MosaicBert  # noqa: E402

dev = "cuda"
BF = torch.bfloat16


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def ln_ablation(T=65536, H=768, n_fwd=25, n_bwd=24):
    g = torch.ones(H, dtype=BF, device=dev)
    b = torch.zeros(H, dtype=BF, device=dev)
    st = torch.empty(T, 2, dtype=torch.float32, device=dev)
    dg, db, ds = (torch.zeros(H, device=dev) for _ in range(3))
    out = {}
    for name, dt in (("bf16", BF), ("fp32", torch.float32)):
        x = torch.randn(T, H, device=dev).to(dt)
        dy = torch.randn(T, H, device=dev).to(dt)
        y, dx = torch.empty_like(x), torch.empty_like(x)
        if dt == BF:
            f = lambda: L.layernorm_forward(x, g, b, 1e-12, y, st)  # noqa: E731
            bw = lambda: L.layernorm_backward(dy, x, st, g, dx, dg, db, ds)  # noqa: E731
        else:
            f = lambda: L.layernorm_forward_f32(x, g, b, 1e-12, y, st)  # noqa: E731
            bw = lambda: L.layernorm_backward_f32(dy, x, st, g, dx, dg, db, ds)  # noqa: E731
        tf, tb = timed(f), timed(bw)
        out[name] = {"fwd_us": tf * 1e3, "bwd_us": tb * 1e3, "per_step_ms": n_fwd * tf + n_bwd * tb}
        del x, dy, y, dx
    out["fp32_over_bf16"] = out["fp32"]["per_step_ms"] / out["bf16"]["per_step_ms"]
    out["note"] = f"{n_fwd} LN forwards + {n_bwd} LN backwards per C2 step (T={T}, H={H})"
    return out


def glu_ablation(T=65536, H=768, I=3072, layers=12):
    X = torch.randn(T, H, device=dev).to(BF)
    W1v = (torch.randn(2 * I, H, device=dev) * 0.02).to(BF)
    b1v = torch.zeros(2 * I, dtype=BF, device=dev)
    W2 = (torch.randn(H, I, device=dev) * 0.02).to(BF)
    dF = torch.randn(T, H, device=dev).to(BF)
    Gd = torch.empty(T, 2 * I, dtype=BF, device=dev)
    Z = torch.empty(T, I, dtype=BF, device=dev)
    dU = torch.empty(T, 2 * I, dtype=BF, device=dev)
    fused_f = timed(lambda: L.geglu_forward(X, W1v, b1v, Gd, Z))
    fused_b = timed(lambda: L.geglu_backward(dF, W2, Gd, dU))
    del Gd, dU
    Ua = torch.empty(T, I, dtype=BF, device=dev)
    Ug = torch.empty(T, I, dtype=BF, device=dev)
    W1, V = W1v[:I], W1v[I:]
    b1, bv = b1v[:I], b1v[I:]
    dZ = torch.empty(T, I, dtype=BF, device=dev)
    dUa, dUg = torch.empty_like(Ua), torch.empty_like(Ug)

    def naive_fwd():
        L.gemm(T, I, H, X, H, 0, W1, H, 0, Ua, I, bias=b1)
        L.gemm(T, I, H, X, H, 0, V, H, 0, Ug, I, bias=bv)
        L.geglu_naive_forward(Ua, Ug, Z)

    def naive_bwd():
        L.gemm(T, I, H, dF, H, 0, W2, I, 1, dZ, I)
        L.geglu_naive_backward(dZ, Ua, Ug, dUa, dUg)

    naive_f, naive_b = timed(naive_fwd), timed(naive_bwd)
    out = {"fused": {"fwd_us": fused_f * 1e3, "bwd_us": fused_b * 1e3, "per_step_ms": layers * (fused_f + fused_b)},
           "naive": {"fwd_us": naive_f * 1e3, "bwd_us": naive_b * 1e3, "per_step_ms": layers * (naive_f + naive_b)},
           "note": "GLU forward (up-projection + GeGLU) and the GeGLU part of its backward (dZ = dF W2 + the "
                   "elementwise gradient); the remaining dX / dW GEMMs are identical in both and excluded"}
    out["naive_over_fused"] = out["naive"]["per_step_ms"] / out["fused"]["per_step_ms"]
    return out


def model_step_ms(dims: ModelDims, batch: dict, steps=6, warm=3, dropout=0.0, padded=False):
    params = synth.make_model_params(synth.Dims(dims.hidden, dims.heads, dims.intermediate, dims.vocab, dims.layers),
                                     0, "bert")
    model = MosaicBert(dims, params, device=dev, dropout=dropout)
    del params
    ids = torch.from_numpy(batch["input_ids"]).to(dev)
    mask = torch.from_numpy(batch["attention_mask"]).to(dev)
    labels = torch.from_numpy(batch["labels"]).to(dev)
    if padded:
        mask = torch.ones_like(mask)
    ms = timed(lambda: model.train_step([(ids, mask, labels)]), reps=steps, warm=warm)
    del model
    torch.cuda.empty_cache()
    return ms


def main():
    res = {"device": torch.cuda.get_device_name(0)}
    res["ln"] = ln_ablation()
    torch.cuda.empty_cache()
    res["glu"] = glu_ablation()
    torch.cuda.empty_cache()
    base = ModelDims(768, 12, 3072, 30528, 12)
    b5 = synth.make_batch("C5", 5555)
    nonpad = int(b5["attention_mask"].sum())
    t_var = model_step_ms(base, b5)
    t_pad = model_step_ms(base, b5, padded=True)
    res["unpad"] = {"varlen_ms": t_var, "padded_ms": t_pad, "non_pad_tokens": nonpad,
                    "padding_fraction": 1.0 - nonpad / b5["attention_mask"].size,
                    "varlen_tok_s": nonpad / t_var * 1e3, "padded_tok_s": nonpad / t_pad * 1e3,
                    "speedup": t_pad / t_var}
    b2 = synth.make_batch("C2", 2222)
    t_v8 = model_step_ms(base, b2)
    t_v2 = model_step_ms(ModelDims(768, 12, 3072, 30522, 12), b2)
    res["vocab"] = {"v30528_ms": t_v8, "v30522_ms": t_v2, "v30522_over_v30528": t_v2 / t_v8}
    t_d = model_step_ms(base, b2, dropout=0.1)
    res["dropout"] = {"p0_ms": t_v8, "p0.1_ms": t_d, "cost": t_d / t_v8 - 1.0}
    line = json.dumps(res)
    print(line, flush=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
