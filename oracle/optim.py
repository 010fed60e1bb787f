"""fp64 oracle for F1: decoupled AdamW and the warmup + linear-decay learning-rate schedule.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper: "Decoupled AdamW", LR 5e-4 (Base) / 2e-4 (Large), betas [0.9, 0.98], eps 1e-6, WD 1e-5,
warmup 6 %, final LR 0.02 LR (Table A1); "warmup + linear decay learning rate
schedule".

Reading R34: "decoupled" weight decay in the sense of Loshchilov & Hutter
(Algorithm 2): the decay is NOT added to the gradient (so Adam's normalisation never sees it) and
it follows the schedule multiplier eta_t = lr_t / lr_peak, not the learning rate itself:

    m <- b1 m + (1 - b1) g ;  v <- b2 v + (1 - b2) g^2 ;  mh = m / (1 - b1^t) ;  vh = v / (1 - b2^t)
    w <- w - lr_t * mh / (sqrt(vh) + eps) - (lr_t / lr_peak) * wd * w

so at the peak rate a step with g = 0 multiplies w by (1 - wd) exactly as SPEC's example
states.  The optimizer is handed wd_step = (lr_t / lr_peak) * wd, the per-step decay factor.
The gradient arrives scaled by grad_scale (1 / N_masked_global, reading R18).  Applied to every
parameter (the paper names no exclusions).
"""
from __future__ import annotations

import numpy as np

__all__ = ["lr_at", "adamw_step"]


def lr_at(step: int, total_steps: int, lr_peak: float, warmup: float = 0.06, final: float = 0.02) -> float:
    """Warmup 6 % then linear decay to 0.02 * lr_peak at total_steps (Table A1):
    linear 0 -> lr_peak over the first warmup*total steps, then linear lr_peak -> final*lr_peak."""
    if not 0 <= step <= total_steps:
        raise ValueError("step outside [0, total_steps]")
    w = warmup * total_steps
    if step <= w:
        return lr_peak * step / w if w > 0 else lr_peak
    frac = (step - w) / (total_steps - w)
    return lr_peak * (1.0 + (final - 1.0) * frac)


def adamw_step(w, m, v, g, t: int, lr: float, wd_step: float, betas=(0.9, 0.98), eps: float = 1e-6,
               grad_scale: float = 1.0):
    """One decoupled-AdamW step (R34) in float64; returns new (w, m, v).  t >= 1 is the step count
    used for bias correction."""
    b1, b2 = betas
    g = np.asarray(g, dtype=np.float64) * grad_scale
    m = b1 * np.asarray(m, dtype=np.float64) + (1.0 - b1) * g
    v = b2 * np.asarray(v, dtype=np.float64) + (1.0 - b2) * g * g
    mh = m / (1.0 - b1 ** t)
    vh = v / (1.0 - b2 ** t)
    w = np.asarray(w, dtype=np.float64)
    w = w - lr * mh / (np.sqrt(vh) + eps) - wd_step * w
    return w, m, v
