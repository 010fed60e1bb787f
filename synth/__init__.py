"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests, smoke() and bench.py.

This module holds NO arithmetic of the method (no attention, GeGLU, LayerNorm, loss ...): only
random-number draws, the bf16 storage rounding of those draws, and the batch/length recipes of
DESIGN.md §"Input recipe".  Both the CUDA path and the fp64 oracle consume exactly the arrays
produced here (the oracle upcasts the same bf16 values to fp64).

Configs follow BASELINE.json ``configs`` (C1..C5) with the per-GPU micro-batch of SURVEY §8.0:
  C1 tiny   H=64  heads=2  I=256  V=128   layers=1  L=16  B=4   (ragged, one l=16 row, one l=1 row)
  C2 Base   H=768 heads=12 I=3072 V=30528 layers=12 L=128 B=512 (all rows full, C4 docs exceed 128)
  C3 Large  H=1024 heads=16 I=4096 V=30528 layers=24 L=128 B=256
  C4 Base seq512  L=512 B=128
  C5 Base high-pad: lengths clip(round(LogNormal(ln(0.42 L), 0.8)), 2, L)  (~50% pad)
"""
from __future__ import annotations

import dataclasses
import numpy as np

IGNORE = -100  # label ignore index
PAD_ID, CLS_ID, SEP_ID, MASK_ID = 0, 101, 102, 103
REAL_VOCAB = 30522  # bert-base-uncased; padded to 30528


@dataclasses.dataclass(frozen=True)
class Dims:
    hidden: int
    heads: int
    intermediate: int
    vocab: int
    layers: int
    ln_eps: float = 1e-12

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    dims: Dims
    seq_len: int
    micro_batch: int
    lengths: str  # "c1" | "full" | "lognormal"


BASE = Dims(768, 12, 3072, 30528, 12)
LARGE = Dims(1024, 16, 4096, 30528, 24)
TINY = Dims(64, 2, 256, 128, 1)

CONFIGS = {
    "C1": Config("C1", TINY, 16, 4, "c1"),
    "C2": Config("C2", BASE, 128, 512, "full"),
    "C3": Config("C3", LARGE, 128, 256, "full"),
    "C4": Config("C4", BASE, 512, 128, "full"),
    "C5": Config("C5", BASE, 128, 512, "lognormal"),
}


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float values to the nearest bfloat16 (RNE) and return them as float32."""
    import torch

    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    return t.to(torch.bfloat16).to(torch.float32).numpy()


def rng_for(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


# ----------------------------------------------------------------------------------------------
# batches
# ----------------------------------------------------------------------------------------------
def make_lengths(kind: str, B: int, L: int, rng: np.random.Generator) -> np.ndarray:
    if kind == "c1":
        lens = rng.integers(1, L + 1, size=B)
        if B >= 1:
            lens[0] = L  # a full row (edge)
        if B >= 2:
            lens[-1] = 1  # a length-1 row (edge)
    elif kind == "full":
        lens = np.full(B, L)
    elif kind == "lognormal":
        lens = np.clip(np.round(rng.lognormal(np.log(0.42 * L), 0.8, size=B)), 2, L)
    elif kind.startswith("uniform"):
        lens = rng.integers(1, L + 1, size=B)
    else:
        raise ValueError(kind)
    return lens.astype(np.int64)


def mask_from_lengths(lens: np.ndarray, L: int) -> np.ndarray:
    return (np.arange(L)[None, :] < np.asarray(lens)[:, None]).astype(np.int32)


def make_batch(cfg: Config | str, seed: int, B: int | None = None, L: int | None = None,
               lengths: np.ndarray | None = None, mlm_ratio: float = 0.3) -> dict:
    """ids / attention_mask / labels for one micro-batch, right-padded.

    MLM: Bernoulli(mlm_ratio) over real non-special positions (reading R19); label = the
    original id, IGNORE elsewhere; masked inputs become [MASK] 80% / random 10% / kept 10%.
    """
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    B = cfg.micro_batch if B is None else B
    L = cfg.seq_len if L is None else L
    V = cfg.dims.vocab
    rng = rng_for(seed)
    lens = make_lengths(cfg.lengths, B, L, rng) if lengths is None else np.asarray(lengths)
    mask = mask_from_lengths(lens, L)
    pos = np.arange(L)[None, :]
    if cfg.lengths == "c1":
        ids = rng.integers(5, V, size=(B, L))
        cand = mask.astype(bool)
        mask_tok = 4
        lo_rand, hi_rand = 5, V
    else:
        ids = rng.integers(1000, REAL_VOCAB, size=(B, L))
        ids[:, 0] = CLS_ID
        ids[np.arange(B), np.maximum(lens - 1, 0)] = SEP_ID
        cand = (pos >= 1) & (pos < (lens[:, None] - 1))
        mask_tok = MASK_ID
        lo_rand, hi_rand = 1000, REAL_VOCAB
    ids = np.where(mask.astype(bool), ids, PAD_ID)
    sel = (rng.random((B, L)) < mlm_ratio) & cand
    labels = np.where(sel, ids, IGNORE)
    u = rng.random((B, L))
    rand_ids = rng.integers(lo_rand, hi_rand, size=(B, L))
    inp = np.where(sel & (u < 0.8), mask_tok, ids)
    inp = np.where(sel & (u >= 0.8) & (u < 0.9), rand_ids, inp)
    return {
        "input_ids": inp.astype(np.int32),
        "attention_mask": mask.astype(np.int32),
        "labels": labels.astype(np.int32),
        "lengths": lens.astype(np.int32),
    }


def make_hidden(mask: np.ndarray, H: int, seed: int, pad_scale: float = 10.0) -> np.ndarray:
    """Padded hidden states [B,L,H] (bf16 values): N(0,1) on real rows, N(0,pad_scale^2) garbage
    on pad rows (exercises pin P9: nothing may leak from pad rows)."""
    rng = rng_for(seed)
    B, L = mask.shape
    x = rng.standard_normal((B, L, H))
    x = np.where(mask[..., None].astype(bool), x, pad_scale * rng.standard_normal((B, L, H)))
    return bf16_round(x)


def make_grad(mask: np.ndarray, H: int, seed: int) -> np.ndarray:
    """Upstream gradient [B,L,H] (bf16 values): N(0,1) on real rows, exactly 0 on pad rows."""
    rng = rng_for(seed)
    B, L = mask.shape
    g = rng.standard_normal((B, L, H)) * mask[..., None]
    return bf16_round(g)


# ----------------------------------------------------------------------------------------------
# parameters (nn.Linear convention W[out, in]; all values bf16-exact float32)
# ----------------------------------------------------------------------------------------------
LAYER_KEYS = ("w_qkv", "b_qkv", "w_o", "b_o", "ln1_g", "ln1_b",
              "w_1v", "b_1v", "w_2", "b_2", "ln2_g", "ln2_b")
HEAD_KEYS = ("w_t", "b_t", "lnh_g", "lnh_b", "b_dec")
EMB_KEYS = ("emb", "type_emb", "lne_g", "lne_b")


def _w(rng, out_f, in_f, regime):
    std = 0.02 if regime == "bert" else 1.0 / np.sqrt(in_f)
    return rng.standard_normal((out_f, in_f)) * std


def _b(rng, n, regime):
    return np.zeros(n) if regime == "bert" else 0.1 * rng.standard_normal(n)


def _g(rng, n, regime):
    return np.ones(n) if regime == "bert" else 1.0 + 0.1 * rng.standard_normal(n)


def make_layer_params(dims: Dims, seed: int, regime: str = "bert") -> dict:
    rng = rng_for(seed)
    H, I = dims.hidden, dims.intermediate
    p = {
        "w_qkv": _w(rng, 3 * H, H, regime), "b_qkv": _b(rng, 3 * H, regime),
        "w_o": _w(rng, H, H, regime), "b_o": _b(rng, H, regime),
        "ln1_g": _g(rng, H, regime), "ln1_b": _b(rng, H, regime),
        "w_1v": _w(rng, 2 * I, H, regime), "b_1v": _b(rng, 2 * I, regime),
        "w_2": _w(rng, H, I, regime), "b_2": _b(rng, H, regime),
        "ln2_g": _g(rng, H, regime), "ln2_b": _b(rng, H, regime),
    }
    return {k: bf16_round(v) for k, v in p.items()}


def make_model_params(dims: Dims, seed: int, regime: str = "bert", n_layers: int | None = None) -> dict:
    n_layers = dims.layers if n_layers is None else n_layers
    rng = rng_for(seed)
    H, V = dims.hidden, dims.vocab
    emb_std = 0.02 if regime == "bert" else 1.0 / np.sqrt(H)
    p = {
        "emb": rng.standard_normal((V, H)) * emb_std,
        "type_emb": rng.standard_normal((2, H)) * emb_std,
        "lne_g": _g(rng, H, regime), "lne_b": _b(rng, H, regime),
        "w_t": _w(rng, H, H, regime), "b_t": _b(rng, H, regime),
        "lnh_g": _g(rng, H, regime), "lnh_b": _b(rng, H, regime),
        "b_dec": _b(rng, V, regime),
    }
    p = {k: bf16_round(v) for k, v in p.items()}
    p["layers"] = [make_layer_params(dims, seed * 1000 + 17 + l, regime) for l in range(n_layers)]
    return p

