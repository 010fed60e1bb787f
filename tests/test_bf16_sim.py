"""Pins of the storage model tests/bf16_sim.py (the tool that derives reading R33's a-priori bar):
with no rounding site it IS the oracle's step (same arithmetic, nothing dropped), with dropout
included, and every site it names is a real rounding point (each one alone moves the result)."""
import numpy as np
import pytest

import bf16_sim as S
import oracle as O
import synth


def _case(seed=5, dims=synth.TINY, n_layers=2):
    params = synth.make_model_params(dims, seed, "stress", n_layers=n_layers)
    batch = synth.make_batch("C1", 100 + seed)
    n_lab = int(((batch["labels"] != -100) & (batch["attention_mask"] != 0)).sum())
    return dims, params, batch, 1.0 / n_lab


@pytest.mark.parametrize("dropout", [None, dict(p=0.3, seed=11)])
def test_no_sites_equals_oracle_step(dropout):
    dims, params, batch, inv = _case()
    loss, grads = O.model_forward_backward(batch, params, O.alibi_slopes(dims.heads), dims.ln_eps, inv, dropout)
    l2, _, _, g2 = S.model_step(batch, params, dims.heads, inv, dims.ln_eps, sites=(), dropout=dropout)
    assert abs(loss - l2) <= 1e-12 * max(1.0, abs(loss))
    flat = lambda g: [g[k] for k in ("emb", "type_emb", "lne_g", "lne_b", "w_t", "b_t", "lnh_g", "lnh_b", "b_dec")] + [  # noqa
        v for lg in g["layers"] for _, v in sorted(lg.items())]
    for a, b in zip(flat(grads), flat(g2)):
        assert np.max(np.abs(a - b)) <= 1e-10 * max(1.0, np.max(np.abs(a)))


def test_dropout_rows_subset_matches_full_batch():
    """dropout['rows'] (the sample's packed rows inside a larger micro-batch) reproduces the masks
    the full batch draws for those rows."""
    mask = synth.mask_from_lengths(np.array([6, 3, 5]), 6)
    full0, full1 = O.dropout_masks(mask, 16, dict(p=0.4, seed=9, stream=2))
    cu = np.concatenate([[0], np.cumsum(mask.sum(1))])
    rows = np.concatenate([np.arange(cu[b], cu[b + 1]) for b in (0, 2)])
    sub0, sub1 = O.dropout_masks(mask[[0, 2]], 16, dict(p=0.4, seed=9, stream=2, rows=rows))
    assert np.array_equal(sub0, full0[[0, 2]]) and np.array_equal(sub1, full1[[0, 2]])


def test_every_site_rounds():
    dims, params, batch, inv = _case(n_layers=1)
    ref = S.model_step(batch, params, dims.heads, inv, dims.ln_eps, sites=())
    for site in sorted(S.ALL):
        out = S.model_step(batch, params, dims.heads, inv, dims.ln_eps, sites={site})
        moved = max(np.max(np.abs(a - b)) for a, b in zip(
            [out[2], out[3]["w_t"], out[3]["emb"], out[3]["layers"][0]["w_qkv"]],
            [ref[2], ref[3]["w_t"], ref[3]["emb"], ref[3]["layers"][0]["w_qkv"]]))
        assert moved > 0.0, site
