"""Derivation of the depth-12/24 parity bar of reading R33.  Run by hand (CPU only):

    python tests/r33_spread.py C2 C5 C3 C4   ->  tests/golden/r33_spread.json

For each config, on the exact sample that tests/test_gpu_fullsize.py::test_model_step_fullsize_sampled
uses (labels only on the sampled sequences), it computes
  * the exact fp64 oracle step (oracle/), and
  * the bf16 STORAGE MODEL (tests/bf16_sim.py, sites = ALL: every tensor the CUDA path stores in
    bf16 is rounded RNE at the place the kernels store it), and R further realisations of it whose
    pre-rounding values carry a 1e-6 relative jitter (the size of fp32 accumulation-order noise
    over K = 768..6144 terms) — i.e. other, equally valid bf16 implementations of the same step.
Per tensor, model(t) = max|model - exact| / max|exact|, and model_worst = max_t model(t).  The GPU
path is one more realisation of that rounding process, so R33's bar for every tensor is
max(2e-2, F x model_worst); F is the largest realisation_worst / model_worst observed here, with a
margin.  (Per-tensor bars F x model(t) need a larger F — the per-tensor max-rel of one realisation is
a noisy statistic — and are reported as factor_needed_per_tensor.)  No GPU output is involved."""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import bf16_sim as S  # noqa: E402
import synth  # noqa: E402
from parity import metrics  # noqa: E402

JITTER = 1e-6


def sample_case(cfg):
    """The sub-batch, parameters and normaliser of test_model_step_fullsize_sampled (part b)."""
    c = synth.CONFIGS[cfg]
    batch = synth.make_batch(cfg, 1000 * int(cfg[1]) + 0, B=c.micro_batch)
    mask, labels = batch["attention_mask"], batch["labels"]
    lens = mask.sum(1)
    samp = sorted({0, len(lens) // 2, len(lens) - 1, int(np.argmin(lens)), int(np.argmax(lens))})
    lab_s = np.full_like(labels, -100)
    lab_s[samp] = labels[samp]
    n_s = int(((lab_s != -100) & (mask != 0)).sum())
    sub = {k: v[samp] for k, v in batch.items()}
    sub["labels"] = lab_s[samp]
    Ls = int(lens[samp].max())
    sub = {k: (v[:, :Ls] if np.ndim(v) == 2 else v) for k, v in sub.items()}
    return c.dims, sub, synth.make_model_params(c.dims, 0, "bert"), 1.0 / n_s


def flat(g):
    out = {k: g[k] for k in ("emb", "type_emb", "lne_g", "lne_b", "w_t", "b_t", "lnh_g", "lnh_b", "b_dec")}
    for li, lg in enumerate(g["layers"]):
        for k, v in lg.items():
            out[f"L{li}.{k}"] = v
    return out


def spread(cfg, R):
    d, sub, params, inv = sample_case(cfg)
    ex = S.model_step(sub, params, d.heads, inv, d.ln_eps, sites=())
    md = S.model_step(sub, params, d.heads, inv, d.ln_eps)
    E, M = flat(ex[3]), flat(md[3])
    m0 = {k: metrics(M[k], E[k])[0] for k in E}
    m0["dX0"] = metrics(md[2], ex[2])[0]
    ratios, worst, need = [], [], 0.0
    for r in range(R):
        jo = S.model_step(sub, params, d.heads, inv, d.ln_eps, jitter=JITTER, seed=r + 1)
        jr = flat(jo[3])
        rr = {k: metrics(jr[k], E[k])[0] for k in E}
        rr["dX0"] = metrics(jo[2], ex[2])[0]
        ratios += [rr[k] / m0[k] for k in rr if m0[k] > 0]
        worst.append(max(rr.values()))
        # the per-tensor rule max(2e-2, F * model(t)) would need this F (only tensors above 2e-2 count)
        need = max([need] + [rr[k] / m0[k] for k in rr if rr[k] > 2e-2])
    q = np.quantile(ratios, [0.5, 0.9, 0.99, 1.0])
    mw = max(m0.values())
    return dict(tensors=len(rr), realisations=R, model_worst=mw, realisation_worst=worst,
                factor_needed=max(w / mw for w in worst), per_tensor_ratio_p50=q[0], per_tensor_ratio_p90=q[1],
                per_tensor_ratio_p99=q[2], per_tensor_ratio_max=q[3], factor_needed_per_tensor=need)


if __name__ == "__main__":
    out_path = os.path.join(HERE, "golden", "r33_spread.json")
    res = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for cfg in sys.argv[1:] or ["C2", "C5", "C3", "C4"]:
        t = time.time()
        res[cfg] = spread(cfg, 6 if cfg in ("C2", "C5") else 4)
        print(cfg, json.dumps(res[cfg]), f"{time.time() - t:.0f}s", flush=True)
        json.dump(res, open(out_path, "w"), indent=1)
