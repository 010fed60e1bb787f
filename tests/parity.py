"""Comparison helpers for GPU-vs-oracle parity (tolerance of BASELINE.json north_star, reading R24):
per tensor max|g - r| / max|r| <= 2e-2 and cosine >= 0.999; loss |delta| <= 1e-2."""
import numpy as np

MAX_REL = 2e-2
MIN_COS = 0.999


def metrics(got, ref):
    g = np.asarray(got, dtype=np.float64).ravel()
    r = np.asarray(ref, dtype=np.float64).ravel()
    denom = max(np.max(np.abs(r)), 1e-30)
    rel = float(np.max(np.abs(g - r)) / denom) if g.size else 0.0
    ng, nr = np.linalg.norm(g), np.linalg.norm(r)
    cos = float(np.dot(g, r) / (ng * nr)) if ng > 0 and nr > 0 else (1.0 if ng == nr else 0.0)
    return rel, cos


def check(name, got, ref, max_rel=MAX_REL, min_cos=MIN_COS):
    rel, cos = metrics(got, ref)
    assert np.all(np.isfinite(np.asarray(got, dtype=np.float64))), f"{name}: non-finite values"
    assert rel <= max_rel and cos >= min_cos, f"{name}: max_rel={rel:.3e} cos={cos:.6f}"
    return rel, cos


def to_dev(a, dtype):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a)).to(dtype).cuda()


def np64(t):
    return t.double().cpu().numpy()
