"""Pins of the fp64 oracle against what the paper and mathematics fix.
None of these compare the oracle with a retyped copy of itself: each uses a printed value, a
closed form, a textbook/library special case, an invariant or brute force."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


# ----------------------------------------------------------------------------- P1 / P2 unpad
def test_p1_unpad_worked_example():
    g = GOLD["unpad_example"]
    cu, idx, mx, st = O.unpad_index(np.array(g["mask"]))
    assert cu.tolist() == g["cu_seqlens"]
    assert idx.tolist() == g["indices"]
    assert mx == g["max_seqlen"] and st == O.MB_OK


def _brute_unpad(mask):
    """Brute force by explicit loops over (b, l): the definition of S:336-341."""
    B, L = mask.shape
    cu, idx, mx = [0], [], 0
    for b in range(B):
        n = 0
        for l in range(L):
            if mask[b, l]:
                idx.append(b * L + l)
                n += 1
        cu.append(cu[-1] + n)
        mx = max(mx, n)
    return cu, idx, mx


@pytest.mark.parametrize("seed", range(6))
def test_p1_unpad_bruteforce(seed):
    rng = np.random.default_rng(seed)
    B, L = rng.integers(1, 9), rng.integers(1, 40)
    lens = rng.integers(0, L + 1, size=B)
    mask = synth.mask_from_lengths(lens, L)
    cu, idx, mx, st = O.unpad_index(mask)
    bcu, bidx, bmx = _brute_unpad(mask)
    assert cu.tolist() == bcu and idx.tolist() == bidx and mx == bmx and st == O.MB_OK
    assert np.all(np.diff(cu) >= 0) and cu[0] == 0 and cu[-1] == len(idx)


def test_p1_nonprefix_rejected():
    mask = np.array([[1, 0, 1, 0], [1, 1, 0, 0]])
    _, idx, _, st = O.unpad_index(mask)
    assert st == O.MB_ERR_MASK_LAYOUT
    assert idx.tolist() == [0, 2, 4, 5]  # indices still = flat nonzero positions


def test_p2_roundtrip_bitwise():
    g = GOLD["unpad_example"]
    mask = np.array(g["mask"])
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 4, 5)).astype(np.float32)
    _, idx, _, _ = O.unpad_index(mask)
    back = O.pad(O.unpad(x, idx), idx, 2, 4)
    assert np.array_equal(back, x * mask[..., None])
    for b, l in g["zero_positions"]:
        assert np.all(back[b, l] == 0)


# ----------------------------------------------------------------------------- P3 / P4 ALiBi
def test_p3_slopes_closed_form():
    assert O.alibi_slopes(8).tolist() == GOLD["alibi_slopes_n8"]["value"]
    s12 = O.alibi_slopes(12)
    g = GOLD["alibi_slopes_n12_first_last"]
    assert abs(s12[0] - g["first"]) < 1e-10 and s12[2] == g["third"] and s12[-1] == g["last"]
    assert O.alibi_slopes(2).tolist() == [0.0625, 0.00390625]
    s16 = O.alibi_slopes(16)
    assert np.allclose(s16, 2.0 ** (-0.5 * np.arange(1, 17)), rtol=0, atol=0)
    for n in (2, 8, 12, 16):
        s = O.alibi_slopes(n)
        assert np.all(np.abs(s[1:] / s[:-1] - 2.0 ** (-8.0 / n)) < 1e-12)  # ratio 2^{-8/n}
        assert abs(s[0] - 2.0 ** (-8.0 / n)) < 1e-15
    with pytest.raises(ValueError):
        O.alibi_slopes(0)


def test_p4_bias_worked_examples():
    assert O.alibi_bias(3, 1.0).tolist() == GOLD["alibi_bias_L3_m1"]["value"]
    assert O.alibi_bias(2, 0.5).tolist() == GOLD["alibi_bias_L2_m05"]["value"]
    b = O.alibi_bias(7, 0.3)
    assert np.array_equal(b, b.T) and np.all(np.diag(b) == 0)


def _qkv(B, L, n, d, seed):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((B, L, n, d)) for _ in range(3)]


def test_p4b_alibi_softmax_closed_form():
    """Q = K = 0 -> weights w_ij = e^{-m|i-j|}/sum_{j'<l} e^{-m|i-j'|} (geometric sum).
    l=2, m=ln 3 -> row 0 = [3/4, 1/4]."""
    B, L, n, d = 2, 6, 1, 4
    q = np.zeros((B, L, n, d))
    k = np.zeros((B, L, n, d))
    v = np.zeros((B, L, n, d))
    v[..., 0] = np.arange(L)[None, :, None]  # value = key position -> output = E_w[j]
    v[..., 1] = 1.0
    mask = synth.mask_from_lengths(np.array([2, 5]), L)
    m = math.log(3.0)
    C, cache = O.attention_forward(q, k, v, mask, np.array([m]))
    P = cache[3]
    assert np.allclose(P[0, 0, 0, :2], [0.75, 0.25], atol=1e-15)
    assert np.allclose(P[0, 0, 1, :2], [0.25, 0.75], atol=1e-15)
    # sequence 1, l=5: closed form per row, positions restart per sequence
    for i in range(L):
        w = np.array([3.0 ** (-abs(i - j)) for j in range(5)])
        w /= w.sum()
        assert np.allclose(P[1, 0, i, :5], w, atol=1e-14)
        assert np.all(P[1, 0, i, 5:] == 0)
        assert abs(C[1, i, 0, 0] - np.dot(w, np.arange(5))) < 1e-13
    assert np.allclose(C[..., 1][mask.astype(bool)], 1.0)


# ----------------------------------------------------------------------------- P5 / P6 torch SDPA
def _torch_sdpa(q, k, v, bias):
    import torch
    import torch.nn.functional as F
    tq, tk, tv = (torch.from_numpy(np.ascontiguousarray(x.transpose(0, 2, 1, 3))) for x in (q, k, v))
    out = F.scaled_dot_product_attention(tq, tk, tv, attn_mask=torch.from_numpy(bias))
    return out.numpy().transpose(0, 2, 1, 3)


@pytest.mark.parametrize("zero_slopes", [True, False])
def test_p5_p6_sdpa_equivalence(zero_slopes):
    B, L, n, d = 3, 11, 4, 8
    q, k, v = _qkv(B, L, n, d, 1)
    lens = np.array([11, 6, 1])
    mask = synth.mask_from_lengths(lens, L)
    slopes = np.zeros(n) if zero_slopes else O.alibi_slopes(n)
    C, _ = O.attention_forward(q, k, v, mask, slopes)
    i = np.arange(L)
    bias = np.zeros((B, n, L, L))
    for h in range(n):
        bias[:, h] = -slopes[h] * np.abs(i[:, None] - i[None, :])
    bias = np.where(mask[:, None, None, :].astype(bool), bias, -np.inf)
    ref = _torch_sdpa(q, k, v, bias)
    real = mask.astype(bool)
    assert np.max(np.abs(C[real] - ref[real])) < 1e-12


# ----------------------------------------------------------------------------- P7 limits
def test_p7_large_slope_identity_and_len1():
    B, L, n, d = 2, 7, 2, 4
    q, k, v = _qkv(B, L, n, d, 2)
    mask = synth.mask_from_lengths(np.array([7, 1]), L)
    C, cache = O.attention_forward(q, k, v, mask, np.array([1e4, 1e4]))
    real = mask.astype(bool)
    assert np.max(np.abs(C[real] - v[real])) < 1e-12
    dC = np.random.default_rng(3).standard_normal(C.shape) * mask[..., None, None]
    dq, dk, dv = O.attention_backward(dC, cache)
    assert np.max(np.abs(dv[real] - dC[real])) < 1e-12
    assert np.max(np.abs(dq)) < 1e-12 and np.max(np.abs(dk)) < 1e-12
    # l = 1 with ordinary slopes: output = V row
    C1, _ = O.attention_forward(q, k, v, mask, O.alibi_slopes(n))
    assert np.max(np.abs(C1[1, 0] - v[1, 0])) < 1e-15


def test_p7_len1_layer():
    """l=1: attention output = v, so A = Wo (Wv x + bv) + bo."""
    dims = synth.TINY
    p = synth.make_layer_params(dims, 5, "stress")
    H = dims.hidden
    x = np.random.default_rng(4).standard_normal((1, 1, H))
    mask = np.ones((1, 1), dtype=np.int32)
    _, c = O.encoder_layer_forward(x, mask, O.alibi_slopes(dims.heads), p)
    wv, bv = p["w_qkv"][2 * H:].astype(np.float64), p["b_qkv"][2 * H:].astype(np.float64)
    A = (x[0, 0] @ wv.T + bv) @ p["w_o"].astype(np.float64).T + p["b_o"]
    assert np.max(np.abs(c["S1"][0, 0] - (A + x[0, 0]))) < 1e-12


# ----------------------------------------------------------------------------- P8 / P9 unpadded == padded
def _layer_case(seed, regime="stress", dims=synth.TINY, lens=(16, 9, 3, 1), L=16):
    p = synth.make_layer_params(dims, seed, regime)
    mask = synth.mask_from_lengths(np.array(lens), L)
    X = synth.make_hidden(mask, dims.hidden, seed + 1)
    dY = synth.make_grad(mask, dims.hidden, seed + 2)
    return p, mask, X, dY


def test_p8_unpadded_equals_padded():
    dims = synth.TINY
    p, mask, X, dY = _layer_case(0)
    slopes = O.alibi_slopes(dims.heads)
    Y, c = O.encoder_layer_forward(X, mask, slopes, p)
    dX, g = O.encoder_layer_backward(dY, c)
    gsum = {k: np.zeros_like(v) for k, v in g.items()}
    for b, lb in enumerate(mask.sum(1)):
        Yb, cb = O.encoder_layer_forward(X[b:b + 1, :lb], np.ones((1, lb)), slopes, p)
        dXb, gb = O.encoder_layer_backward(dY[b:b + 1, :lb], cb)
        assert np.max(np.abs(Yb[0] - Y[b, :lb])) < 1e-12
        assert np.max(np.abs(dXb[0] - dX[b, :lb])) < 1e-12
        for k in gsum:
            gsum[k] += gb[k]
    for k in g:
        assert np.max(np.abs(gsum[k] - g[k])) < 1e-10 * max(1.0, np.max(np.abs(g[k])))


def test_p9_no_pad_leak():
    dims = synth.TINY
    p, mask, X, dY = _layer_case(1)
    slopes = O.alibi_slopes(dims.heads)
    Y, c = O.encoder_layer_forward(X, mask, slopes, p)
    dX, g = O.encoder_layer_backward(dY, c)
    X2 = X.copy()
    X2[~mask.astype(bool)] = 1e3 * np.random.default_rng(9).standard_normal(X2[~mask.astype(bool)].shape)
    Y2, c2 = O.encoder_layer_forward(X2, mask, slopes, p)
    dX2, g2 = O.encoder_layer_backward(dY, c2)
    real = mask.astype(bool)
    assert np.array_equal(Y[real], Y2[real])
    assert np.array_equal(dX, dX2)
    for k in g:
        assert np.allclose(g[k], g2[k], rtol=0, atol=1e-12 * max(1, np.abs(g[k]).max())), k


def test_p9b_key_bias_gradient_vanishes():
    """Invariant (R31): a key-projection bias adds q_i.b_k/sqrt(d) to every score of query row i —
    a per-row constant the row softmax of Eq. 1 cancels — so dL/db_k = 0 while db_q, db_v do not
    vanish.  Pins the oracle's attention backward (a wrong dS sign/D term breaks the zero rowsum)."""
    dims = synth.TINY
    p, mask, X, dY = _layer_case(2)
    H = dims.hidden
    _, c = O.encoder_layer_forward(X, mask, O.alibi_slopes(dims.heads), p)
    _, g = O.encoder_layer_backward(dY, c)
    db = g["b_qkv"]
    scale = np.max(np.abs(db))
    assert scale > 1e-3
    assert np.max(np.abs(db[H:2 * H])) < 1e-12 * scale
    assert np.max(np.abs(db[:H])) > 1e-3 * scale and np.max(np.abs(db[2 * H:])) > 1e-3 * scale
    # and the key bias leaves the forward unchanged (the reason the gradient vanishes)
    p2 = dict(p)
    p2["b_qkv"] = p["b_qkv"].copy()
    p2["b_qkv"][H:2 * H] += np.random.default_rng(4).standard_normal(H)
    Y1, _ = O.encoder_layer_forward(X, mask, O.alibi_slopes(dims.heads), p)
    Y2, _ = O.encoder_layer_forward(X, mask, O.alibi_slopes(dims.heads), p2)
    real = mask.astype(bool)
    assert np.max(np.abs(Y1[real] - Y2[real])) < 1e-10


# ----------------------------------------------------------------------------- P10 GeGLU
def test_p10_gelu_value():
    assert abs(O.gelu(1.0) - GOLD["gelu_1"]["value"]) < 1e-15
    assert O.gelu(0.0) == 0.0 and abs(O.gelu(10.0) - 10.0) < 1e-6
    x = np.linspace(-4, 4, 17)
    fd = (O.gelu(x + 1e-6) - O.gelu(x - 1e-6)) / 2e-6
    assert np.max(np.abs(fd - O.gelu_grad(x))) < 1e-8


def test_p10_geglu_special_cases():
    dims = synth.TINY
    H, I = dims.hidden, dims.intermediate
    p = synth.make_layer_params(dims, 3, "stress")
    rng = np.random.default_rng(0)
    y1 = rng.standard_normal((5, H))
    # x=0 with zero biases -> GeGLU output 0
    U = np.zeros((5, H)) @ p["w_1v"].T
    assert np.all(O.gelu(U[:, :I]) * U[:, I:] == 0)
    # gate W_V = 0, b_V = 1 -> plain GeLU MLP: run through the layer and compare F
    q = dict(p)
    q["w_1v"] = p["w_1v"].copy(); q["w_1v"][I:] = 0
    q["b_1v"] = p["b_1v"].copy(); q["b_1v"][I:] = 1
    mask = np.ones((1, 5), dtype=np.int32)
    _, c = O.encoder_layer_forward(y1[None], mask, O.alibi_slopes(dims.heads), q)
    Y1 = c["Y1"][0]
    F_plain = O.gelu(Y1 @ p["w_1v"][:I].T + p["b_1v"][:I]) @ p["w_2"].T + p["b_2"]
    assert np.max(np.abs((c["S2"][0] - Y1) - F_plain)) < 1e-12
    # fused == naive split: W1 || V as one GEMM then slice
    _, c = O.encoder_layer_forward(y1[None], mask, O.alibi_slopes(dims.heads), p)
    Y1 = c["Y1"][0]
    W1, Vg = p["w_1v"][:I].astype(np.float64), p["w_1v"][I:].astype(np.float64)
    naive = O.gelu(Y1 @ W1.T + p["b_1v"][:I]) * (Y1 @ Vg.T + p["b_1v"][I:])
    assert np.max(np.abs(naive - c["Z"][0])) < 1e-12


# ----------------------------------------------------------------------------- P11 LayerNorm
def test_p11_layernorm():
    H = 16
    g = np.random.default_rng(0).standard_normal(H)
    b = np.random.default_rng(1).standard_normal(H)
    y, _ = O.layer_norm(np.full((3, H), 2.5), g, b, 1e-12)
    assert np.array_equal(y, np.broadcast_to(b, (3, H)))  # constant row -> beta exactly
    y, _ = O.layer_norm(np.array([[1.0, -1.0]]), np.ones(2), np.zeros(2), 1e-12)
    assert np.allclose(y, np.array([[1, -1]]) / np.sqrt(1 + 1e-12), atol=1e-15)
    v = np.random.default_rng(2).standard_normal((7, H)) * 3 + 1
    y, cache = O.layer_norm(v, g, b, 1e-5)
    xhat, r = cache
    assert np.allclose(xhat.mean(-1), 0, atol=1e-14) and np.allclose((xhat ** 2).mean(-1) * (1 + 1e-5 * r[:, 0] ** 2), 1, atol=1e-12)
    dy = np.random.default_rng(3).standard_normal((7, H))
    dv, dg, db = O.layer_norm_backward(dy, cache, g)
    assert np.max(np.abs(dv.sum(-1))) < 1e-12  # sum_k dv_k = 0
    # sum_k dv_k xhat_k = r * sum(g xhat) * eps / (sigma^2 + eps)  (~0)
    var = 1.0 / r[:, 0] ** 2 - 1e-5
    lhs = (dv * xhat).sum(-1)
    rhs = r[:, 0] * ((dy * g) * xhat).mean(-1) * H * 1e-5 / (var + 1e-5)
    assert np.max(np.abs(lhs - rhs)) < 1e-10


def test_p11_bf16_ln_within_001():
    """bf16 storage of x/gamma/beta/y with fp32 statistics stays within 0.01 of fp32 LN."""
    import torch
    x = torch.randn(2000, 768)
    xb = x.bfloat16().float()
    ref = torch.nn.functional.layer_norm(x, (768,), eps=1e-12)
    y = torch.nn.functional.layer_norm(xb, (768,), eps=1e-12).bfloat16().float()
    assert (y - ref).abs().max().item() <= 0.01 + 2 ** -7 * 4
    yo, _ = O.layer_norm(xb.double().numpy(), np.ones(768), np.zeros(768), 1e-12)
    assert np.max(np.abs(yo - ref.double().numpy())) <= 0.05


# ----------------------------------------------------------------------------- P12 CE
@pytest.mark.parametrize("V", [128, 30528])
def test_p12_ce_zero_decoder(V):
    H = 16
    B, L = 3, 8
    rng = np.random.default_rng(0)
    Y = rng.standard_normal((B, L, H))
    labels = np.full((B, L), O.IGNORE)
    labels[0, 1], labels[1, 2], labels[2, 5], labels[0, 4] = 7, 7, 3, 99
    mask = np.ones((B, L), dtype=np.int32)
    hp = {"w_t": rng.standard_normal((H, H)), "b_t": rng.standard_normal(H),
          "lnh_g": np.ones(H), "lnh_b": np.zeros(H), "b_dec": np.zeros(V)}
    emb = np.zeros((V, H))
    nm = 4
    loss, dY, g, lse = O.mlm_head_forward_backward(Y, labels, mask, hp, emb, 1.0 / nm)
    key = "V30528" if V == 30528 else "V128"
    assert abs(loss - GOLD["ce_zero_decoder_lnV"][key]) < 1e-12
    assert abs(loss - math.log(V)) < 1e-12
    hist = np.bincount([7, 7, 3, 99], minlength=V)
    assert np.max(np.abs(g["b_dec"] - (nm / V - hist) / nm)) < 1e-15
    assert np.all(dY == 0)  # E = 0 -> no gradient reaches the encoder


# ----------------------------------------------------------------------------- P15 / P16 accounting
def test_p15_param_counts():
    base = O.param_count(768, 12, 3072, 30528, 12)
    large = O.param_count(1024, 16, 4096, 30528, 24)
    assert base == 137_474_112 and abs(base / 1e6 - 137) / 137 < 0.01
    assert large == 435_417_920 and abs(large / 1e6 - 430) / 430 < 0.02
    bert = O.param_count(768, 12, 3072, 30522, 12, glu=False, position_rows=512)
    assert abs(bert / 1e6 - 110) / 110 < 0.01
    assert O.param_count(64, 2, 256, 128, 1) == 79_488
    # the synthetic parameter set has exactly these shapes
    p = synth.make_model_params(synth.TINY, 0)
    n = sum(v.size for k, v in p.items() if k != "layers") + sum(v.size for l in p["layers"] for v in l.values())
    assert n == 79_488
    assert GOLD["vocab_round"]["to"] == 64 * math.ceil(GOLD["vocab_round"]["from"] / 64)


def test_p16_mfu_table_h1():
    for row in GOLD["table_h1"]["rows"]:
        got = 100 * O.mfu(row["tok_s"], row["params"], row["gpus"], 312e12)
        assert abs(got - row["mfu_pct"]) < 0.2, row
    bad = GOLD["table_h1"]["inconsistent_row"]
    got = 100 * O.mfu(bad["tok_s"], bad["params"], bad["gpus"], 312e12)
    assert abs(got - 36.2) < 0.1 and abs(got - bad["mfu_pct"]) > 3  # R26: printed row inconsistent


def test_bf16_round_golden():
    assert synth.bf16_round(np.array([0.1]))[0] == GOLD["bf16_round_0p1"]["value"]
    assert np.allclose(O.softmax(np.array([0.0, math.log(3.0)])), GOLD["softmax_0_ln3"]["value"], atol=1e-16)
