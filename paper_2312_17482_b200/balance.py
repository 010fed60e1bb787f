"""Data-parallel shard balancing for ragged batches ("for C5, re-partition by greedy
longest-processing-time bin packing on l_b so per-rank nnz differs by < 0.5 %").

Sequences are independent (attention never crosses cu_seqlens), so any assignment of a
global batch's sequences to ranks computes the same optimizer step; only the per-rank work — the
non-pad token count nnz (GEMMs, LayerNorm, head) and sum l^2 (attention) — depends on it, and the
slowest rank paces every step.  Host-side batch preparation, no device work.
"""
from __future__ import annotations

import heapq

import numpy as np


def lpt_partition(lengths, parts: int, equal_counts: bool = True) -> list[np.ndarray]:
    """Longest-processing-time greedy: sequences in decreasing length, each to the part with the
    smallest token total so far (ties: lower part index).  equal_counts: every part receives
    exactly len(lengths) / parts sequences (requires divisibility), so micro-batch shapes stay the
    same on every rank.  Returns per-part index arrays in increasing order."""
    lengths = np.asarray(lengths, dtype=np.int64)
    n = len(lengths)
    if parts < 1:
        raise ValueError("parts must be >= 1")
    if equal_counts and n % parts:
        raise ValueError("equal_counts needs len(lengths) divisible by parts")
    cap = n // parts if equal_counts else n
    order = np.argsort(-lengths, kind="stable")
    heap = [(0, p) for p in range(parts)]  # (tokens, part)
    count = [0] * parts
    out = [[] for _ in range(parts)]
    for i in order:
        tok, p = heapq.heappop(heap)
        out[p].append(int(i))
        count[p] += 1
        if count[p] < cap:  # a full part leaves the heap for good
            heapq.heappush(heap, (tok + int(lengths[i]), p))
    return [np.sort(np.asarray(o, dtype=np.int64)) for o in out]


def imbalance(lengths, partition) -> float:
    """max part token total / mean part token total - 1."""
    lengths = np.asarray(lengths, dtype=np.int64)
    tot = np.array([lengths[p].sum() for p in partition], dtype=np.float64)
    return float(tot.max() / tot.mean() - 1.0) if tot.mean() > 0 else 0.0
