"""Counter-based Philox-4x32-10 generator and the F2 dropout mask, in plain numpy.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper applies dropout 0.1 to the feed-forward layers but fixes no generator.  Reading
R32: every dropout decision is a pure function of (seed, stream, site, packed row t,
feature f) drawn from Philox-4x32-10 (Salmon, Moraes, Dror & Shaw, "Parallel random numbers: as
easy as 1, 2, 3", SC'11 — the generator behind cuRAND/PyTorch dropout), so the oracle can
regenerate exactly the mask the kernels use:

    counter = (f >> 3, t, 2*stream + site, 0),  key = (seed mod 2^32, seed >> 32)
    w = Philox4x32_10(counter, key)                   (4 x 32-bit words -> 8 features)
    u = 16-bit field (f & 1) of word (f & 7) >> 1     (uniform on 0..65535)
    keep(t, f) = u >= thr = round(p * 65536);  dropout(v) = v * keep * 65536 / (65536 - thr)

The rescale is 1 / P(keep) for u uniform on 0..65535 (inverted dropout: E[dropout(v)] = v); it
equals 1 / (1 - p) exactly when 65536 p is an integer.

site 0 = attention output projection (A6), site 1 = FFN down-projection (A9).
"""
from __future__ import annotations

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57  # Philox-4x32 multipliers (Salmon et al., Table 2)
W0, W1 = 0x9E3779B9, 0xBB67AE85  # Weyl key increments (golden ratio, sqrt(3) - 1)
MASK32 = 0xFFFFFFFF


def philox4x32(ctr, key, rounds: int = 10):
    """ctr uint32[..., 4], key uint32[..., 2] -> uint32[..., 4].  One round:
        (hi0, lo0) = M0 * c0,  (hi1, lo1) = M1 * c2          (64-bit products)
        c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
    with the key bumped by (W0, W1) before every round but the first."""
    c = np.array(ctr, dtype=np.uint64) & MASK32
    k = np.array(key, dtype=np.uint64) & MASK32
    c0, c1, c2, c3 = (c[..., i] for i in range(4))
    k0, k1 = k[..., 0], k[..., 1]
    for r in range(rounds):
        if r:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
        p0 = np.uint64(M0) * c0
        p1 = np.uint64(M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(MASK32)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(MASK32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return np.stack([c0, c1, c2, c3], axis=-1).astype(np.uint32)


def dropout_threshold(p: float) -> int:
    """16-bit drop threshold: an element is dropped iff its uniform u < round(p * 65536)."""
    if not 0.0 <= p < 1.0:
        raise ValueError("dropout p must be in [0, 1)")
    return int(round(p * 65536.0))


def dropout_scale(p: float) -> float:
    """Inverted-dropout rescale 1 / P(keep) = 65536 / (65536 - thr) (so E[keep * scale] = 1)."""
    return 65536.0 / (65536.0 - dropout_threshold(p))


def dropout_keep(T: int, H: int, p: float, seed: int, stream: int, site: int, rows=None) -> np.ndarray:
    """bool [T, H]: keep(t, f) for packed rows t = 0..T-1 (or t = rows[i], i < T, when the rows are
    a subset of a larger packed stream) and features f = 0..H-1 (R32)."""
    thr = dropout_threshold(p)
    t = (np.arange(T, dtype=np.uint64) if rows is None else np.asarray(rows, dtype=np.uint64))[:, None]
    fb = np.arange((H + 7) // 8, dtype=np.uint64)[None, :]
    ctr = np.stack(np.broadcast_arrays(fb, t, np.uint64(2 * stream + site), np.uint64(0)), axis=-1)
    key = np.array([seed & MASK32, (seed >> 32) & MASK32], dtype=np.uint64)
    w = philox4x32(ctr, np.broadcast_to(key, ctr.shape[:-1] + (2,)))  # [T, H/8, 4]
    u = np.stack([w & 0xFFFF, w >> 16], axis=-1).reshape(T, -1)[:, :H]  # feature order 8j+2i+h
    return u >= thr
