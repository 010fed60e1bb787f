"""Deterministic reductions (MB_FLAG_DETERMINISTIC; SURVEY §8a E6 "split-K partials reduced
deterministically", A7 "per-CTA fp32 partials + a deterministic second pass"): two identical steps
give bitwise-identical gradients — for every parameter tensor, at full size — and the deterministic
mode stays within the north_star bar of the oracle.  The default (atomic) mode is only equal up to fp32
reassociation; its run-to-run spread is printed for reference."""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from parity import check, to_dev

pytestmark = pytest.mark.gpu
mb = pytest.importorskip("paper_2312_17482_b200")
from paper_2312_17482_b200 import _lib as L  # noqa: E402

I32 = torch.int32


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mb.lib()


def _grads(model):
    return [b.g.clone() for b in model.buckets]


def _named(model):
    out = {}
    for i, b in enumerate(model.layer_buckets):
        out.update({f"L{i}.{k}": v.clone() for k, v in b.gv.items()})
    for b in (model.head_bucket, model.emb_bucket):
        out.update({k: v.clone() for k, v in b.gv.items()})
    return out


def _two_steps(cfg, n_layers, deterministic, B=None, dropout=0.0):
    c = synth.CONFIGS[cfg]
    d = c.dims
    params = synth.make_model_params(d, 0, "bert", n_layers=n_layers)
    batch = synth.make_batch(cfg, 1000 * int(cfg[1]) + 7, B=B or c.micro_batch)
    model = mb.MosaicBert(mb.ModelDims(d.hidden, d.heads, d.intermediate, d.vocab, n_layers, d.ln_eps), params,
                          deterministic=deterministic, dropout=dropout)
    dev = tuple(to_dev(batch[k], I32) for k in ("input_ids", "attention_mask", "labels"))
    out, named = [], []
    for _ in range(2):
        model.zero_grad()
        model.micro_step(*dev, inv_norm=1.0, drop_seed=99)
        torch.cuda.synchronize()
        out.append(_grads(model))
        named.append(_named(model))
    diff = [k for k in named[0] if not torch.equal(named[0][k], named[1][k])]
    print(f"{cfg} deterministic={deterministic}: tensors differing between two identical steps: {diff}")
    return out


@pytest.mark.parametrize("cfg,n_layers,dropout", [("C2", 12, 0.0), ("C5", 2, 0.1), ("C4", 2, 0.0), ("C3", 1, 0.0)])
def test_deterministic_mode_bitwise_identical(cfg, n_layers, dropout):
    """Full-size micro-batches (C2: the bench's 12-layer Base step; C5 ragged with F2 dropout; C4 the
    l = 512 path with the per-key-tile dQ slabs; C3 Large widths): every gradient bucket — all layers,
    the MLM head, the embedding table (the deterministic scatter) — is bitwise identical over two
    identical steps."""
    g1, g2 = _two_steps(cfg, n_layers, True, dropout=dropout)
    for i, (a, b) in enumerate(zip(g1, g2)):
        assert torch.equal(a, b), f"bucket {i} differs between two identical deterministic steps"
    assert all(float(a.abs().max()) > 0 for a in g1)


def test_default_mode_close_to_deterministic():
    """The atomic default and the deterministic mode compute the same sums in different orders (and
    the deterministic db_qkv sums the stored bf16 dQ/dV columns rather than their fp32 values): per
    bucket they agree far inside the north_star bar; the default's own run-to-run spread is printed."""
    d1, _ = _two_steps("C5", 2, True)
    a1, a2 = _two_steps("C5", 2, False)
    spread = max(float((x - y).abs().max() / max(float(y.abs().max()), 1e-30)) for x, y in zip(a1, a2))
    print(f"default mode run-to-run max-rel spread: {spread:.3e}")
    worst = 0.0
    for x, y in zip(d1, a1):
        rel = float((x - y).abs().max()) / max(float(y.abs().max()), 1e-30)
        cos = float(torch.nn.functional.cosine_similarity(x.double(), y.double(), dim=0))
        worst = max(worst, rel)
        assert rel <= 1e-3 and cos >= 0.99999, (rel, cos)
    print(f"deterministic vs default worst bucket max-rel {worst:.3e}")


def test_deterministic_mode_oracle_parity():
    """The deterministic mode against the fp64 oracle at C1 (stress weights): the north_star bar."""
    dims = synth.TINY
    params = synth.make_model_params(dims, 3, "stress")
    batch = synth.make_batch("C1", 5)
    n_lab = int(((batch["labels"] != -100) & (batch["attention_mask"] != 0)).sum())
    model = mb.MosaicBert(mb.ModelDims(dims.hidden, dims.heads, dims.intermediate, dims.vocab, 1, dims.ln_eps), params,
                          deterministic=True)
    dev = tuple(to_dev(batch[k], I32) for k in ("input_ids", "attention_mask", "labels"))
    model.zero_grad()
    model.micro_step(*dev, inv_norm=1.0 / n_lab)
    torch.cuda.synchronize()
    loss = float(model.loss_sum.item())
    oloss, og = O.model_forward_backward(batch, params, O.alibi_slopes(dims.heads))
    assert abs(loss - oloss) <= 1e-2
    g = model.grads_numpy()
    for k in ("emb", "type_emb", "lne_g", "lne_b", "w_t", "b_t", "lnh_g", "lnh_b", "b_dec"):
        check(f"det.d{k}", g[k], og[k])
    for k, r in og["layers"][0].items():
        check(f"det.L0.d{k}", g["layers"][0][k], r)


def test_deterministic_long_ragged_bitwise():
    """The long-sequence attention backward (decoupled epilogue warpgroup, per-key-tile dQ slabs) in
    deterministic mode on a ragged batch with 1 <= l <= 512 (partial query / key quarters, several
    work units per CTA): two identical steps give bitwise-identical gradients."""
    c = synth.CONFIGS["C4"]
    d = c.dims
    params = synth.make_model_params(d, 0, "bert", n_layers=1)
    rng = np.random.default_rng(5)
    lens = rng.integers(1, 513, size=96)
    lens[:5] = [512, 129, 128, 1, 257]
    batch = synth.make_batch("C4", 4711, B=96, lengths=lens)
    model = mb.MosaicBert(mb.ModelDims(d.hidden, d.heads, d.intermediate, d.vocab, 1, d.ln_eps), params,
                          deterministic=True)
    dev = tuple(to_dev(batch[k], I32) for k in ("input_ids", "attention_mask", "labels"))
    named = []
    for _ in range(2):
        model.zero_grad()
        model.micro_step(*dev, inv_norm=1.0)
        torch.cuda.synchronize()
        named.append(_named(model))
    diff = [k for k in named[0] if not torch.equal(named[0][k], named[1][k])]
    assert not diff, diff
    assert all(torch.isfinite(v).all() for v in named[0].values())
