"""Pins for the oracle's F2 dropout ("0.1 dropout to the feedforward layers"; generator and
placement per reading R32): Philox-4x32-10 against the published Random123 known-answer vectors,
the drop rate, p = 0 as the identity, and finite differences of the layer backward with a fixed
mask (the S:74 metric)."""
import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle as O
import synth
from oracle.philox import dropout_keep, dropout_threshold, philox4x32

GOLD = json.loads((Path(__file__).parent / "golden" / "philox_kat.json").read_text())


@pytest.mark.parametrize("case", range(3))
def test_philox_known_answers(case):
    v = GOLD["philox4x32_10"][case]
    h = lambda xs: np.array([int(x, 16) for x in xs], dtype=np.uint64)  # noqa: E731
    out = philox4x32(h(v["ctr"]), h(v["key"]))
    assert [f"{int(x):08x}" for x in out] == v["out"]


def test_drop_rate_and_threshold():
    assert dropout_threshold(0.1) == 6554 and dropout_threshold(0.0) == 0
    T, H = 2048, 768
    for p in (0.1, 0.5):
        keep = dropout_keep(T, H, p, seed=1234, stream=3, site=1)
        q = dropout_threshold(p) / 65536.0
        n = keep.size
        dropped = n - int(keep.sum())
        assert abs(dropped - q * n) < 5 * math.sqrt(n * q * (1 - q)), (p, dropped / n)
    assert dropout_keep(T, H, 0.0, seed=1, stream=0, site=0).all()


def test_sites_streams_seeds_independent():
    T, H = 512, 256
    base = dropout_keep(T, H, 0.5, seed=7, stream=0, site=0)
    for other in (dropout_keep(T, H, 0.5, seed=7, stream=0, site=1), dropout_keep(T, H, 0.5, seed=7, stream=1, site=0),
                  dropout_keep(T, H, 0.5, seed=8, stream=0, site=0)):
        agree = float((base == other).mean())
        assert abs(agree - 0.5) < 0.01
    # a pure function of (seed, stream, site, t, f): a prefix of rows / features is a sub-block
    assert np.array_equal(dropout_keep(100, 40, 0.5, seed=7, stream=0, site=0), base[:100, :40])


def _layer_case(seed):
    dims = synth.TINY
    p = {k: v.astype(np.float64) for k, v in synth.make_layer_params(dims, seed, "stress").items()}
    mask = synth.mask_from_lengths(np.array([16, 9, 3, 1]), 16)
    X = synth.make_hidden(mask, dims.hidden, seed + 1).astype(np.float64)
    R = synth.make_grad(mask, dims.hidden, seed + 2).astype(np.float64)
    return dims, p, mask, X, R


def test_p0_is_identity():
    dims, p, mask, X, R = _layer_case(3)
    sl = O.alibi_slopes(dims.heads)
    Y0, c0 = O.encoder_layer_forward(X, mask, sl, p)
    Y1, c1 = O.encoder_layer_forward(X, mask, sl, p, dropout=dict(p=0.0, seed=5, stream=0))
    assert np.array_equal(Y0, Y1)
    d0, g0 = O.encoder_layer_backward(R, c0)
    d1, g1 = O.encoder_layer_backward(R, c1)
    assert np.array_equal(d0, d1) and all(np.array_equal(g0[k], g1[k]) for k in g0)


def test_dropout_layer_fd_and_mask_effect():
    dims, p, mask, X, R = _layer_case(5)
    sl = O.alibi_slopes(dims.heads)
    drop = dict(p=0.3, seed=99, stream=2)
    rng = np.random.default_rng(0)

    def f():
        Y, _ = O.encoder_layer_forward(X, mask, sl, p, dropout=drop)
        return float(np.sum(Y * R))

    Y, c = O.encoder_layer_forward(X, mask, sl, p, dropout=drop)
    Yn, _ = O.encoder_layer_forward(X, mask, sl, p)
    real = mask.astype(bool)
    assert np.max(np.abs(Y[real] - Yn[real])) > 1e-2  # the mask changes the output
    dX, g = O.encoder_layer_backward(R, c)
    worst = 0.0
    real_idx = np.argwhere(real)
    for b, l in real_idx[rng.choice(len(real_idx), 12)]:
        for h in rng.choice(dims.hidden, 2):
            ix = (int(b), int(l), int(h))
            old = X[ix]
            X[ix] = old + 1e-5; fp = f()
            X[ix] = old - 1e-5; fm = f()
            X[ix] = old
            fd = (fp - fm) / 2e-5
            worst = max(worst, abs(dX[ix] - fd) / max(1.0, abs(fd)))
    for k in ("w_o", "b_o", "w_2", "b_2", "w_1v"):
        for ix in [np.unravel_index(i, p[k].shape) for i in rng.choice(p[k].size, 8, replace=False)]:
            old = p[k][ix]
            p[k][ix] = old + 1e-5; fp = f()
            p[k][ix] = old - 1e-5; fm = f()
            p[k][ix] = old
            fd = (fp - fm) / 2e-5
            worst = max(worst, abs(g[k][ix] - fd) / max(1.0, abs(fd)))
    assert worst < 1e-6, worst


def test_dropout_scale_is_inverse_keep_probability():
    """Inverted dropout (R32): a kept value is scaled by 1 / P(keep), P(keep) = (65536 - thr) / 65536
    for a uniform 16-bit u, so E[drop(v)] = v for every p; equal to 1 / (1 - p) when 65536 p is an
    integer (p = 1/2, 1/4), and 65536 / 58982 (not 1 / 0.9) at the paper's p = 0.1."""
    from oracle.philox import dropout_scale
    assert dropout_scale(0.5) == 2.0 and dropout_scale(0.25) == 65536.0 / 49152.0
    assert dropout_scale(0.1) == 65536.0 / 58982.0 and dropout_scale(0.0) == 1.0
    u = np.arange(65536)
    for p in (0.1, 0.3, 1.0 / 3.0):
        assert abs(float(np.sum(u >= dropout_threshold(p))) * dropout_scale(p) - 65536.0) < 1e-9
    # the oracle layer applies exactly keep * scale
    mask = synth.mask_from_lengths(np.array([5, 3]), 5)
    D0, _ = O.dropout_masks(mask, 16, dict(p=0.1, seed=3, stream=0))
    vals = np.unique(D0[mask.astype(bool)])
    assert set(vals.tolist()) <= {0.0, 65536.0 / 58982.0}
