"""P13 (finite differences) and P14 (an independent torch-CPU-fp64 autograd implementation) for
the oracle's analytic backward.  Error metric of S:74: |a - fd| / max(1, |fd|)."""
import math

import numpy as np
import pytest

import oracle as O
import synth


def _fd_check(f, x, analytic, idxs, eps=1e-5, tol=1e-6):
    worst = 0.0
    for ix in idxs:
        old = x[ix]
        x[ix] = old + eps
        fp = f()
        x[ix] = old - eps
        fm = f()
        x[ix] = old
        fd = (fp - fm) / (2 * eps)
        worst = max(worst, abs(analytic[ix] - fd) / max(1.0, abs(fd)))
    assert worst < tol, worst
    return worst


def _sample(shape, k, rng, rows=None):
    flat = rng.choice(int(np.prod(shape)), size=min(k, int(np.prod(shape))), replace=False)
    return [np.unravel_index(i, shape) for i in flat]


@pytest.mark.parametrize("regime", ["stress", "bert"])
def test_p13_layer_fd(regime):
    dims = synth.TINY
    rng = np.random.default_rng(0)
    p = {k: v.astype(np.float64) for k, v in synth.make_layer_params(dims, 7, regime).items()}
    mask = synth.mask_from_lengths(np.array([16, 9, 3, 1]), 16)
    X = synth.make_hidden(mask, dims.hidden, 8).astype(np.float64)
    R = synth.make_grad(mask, dims.hidden, 9).astype(np.float64)
    slopes = O.alibi_slopes(dims.heads)

    def f():
        Y, _ = O.encoder_layer_forward(X, mask, slopes, p)
        return float(np.sum(Y * R))

    Y, c = O.encoder_layer_forward(X, mask, slopes, p)
    dX, g = O.encoder_layer_backward(R, c)
    real = np.argwhere(mask.astype(bool))
    xi = [(int(b), int(l), int(h)) for b, l in real[rng.choice(len(real), 20)] for h in rng.choice(dims.hidden, 2)]
    _fd_check(f, X, dX, xi)
    for k in p:
        _fd_check(f, p[k], g[k], _sample(p[k].shape, 24, rng))


def test_p13_model_fd():
    dims = synth.TINY
    rng = np.random.default_rng(1)
    params = synth.make_model_params(dims, 3, "stress")
    params = {k: (v.astype(np.float64) if k != "layers" else [{kk: vv.astype(np.float64) for kk, vv in l.items()} for l in v]) for k, v in params.items()}
    batch = synth.make_batch("C1", 11)
    slopes = O.alibi_slopes(dims.heads)

    def f():
        return O.model_forward_backward(batch, params, slopes)[0]

    loss, grads = O.model_forward_backward(batch, params, slopes)
    assert np.isfinite(loss)
    used = np.unique(batch["input_ids"][batch["attention_mask"].astype(bool)])
    ei = [(int(i), int(h)) for i in rng.choice(used, 10) for h in rng.choice(dims.hidden, 2)]
    ei += [(int(i), int(h)) for i in rng.choice(dims.vocab, 6) for h in rng.choice(dims.hidden, 2)]
    _fd_check(f, params["emb"], grads["emb"], ei)
    for k in ("type_emb", "lne_g", "lne_b", "w_t", "b_t", "lnh_g", "lnh_b", "b_dec"):
        _fd_check(f, params[k], grads[k], _sample(params[k].shape, 12, rng))
    lp, lg = params["layers"][0], grads["layers"][0]
    for k in ("w_qkv", "b_1v", "ln2_g"):
        _fd_check(f, lp[k], lg[k], _sample(lp[k].shape, 8, rng))


# ----------------------------------------------------------------------------- P14 torch autograd
def _torch_layer(X, mask, slopes, p, eps):
    import torch
    import torch.nn.functional as F
    B, L, H = X.shape
    n = len(slopes)
    d = H // n
    qkv = F.linear(X, p["w_qkv"], p["b_qkv"])
    q, k, v = qkv.split(H, dim=-1)
    sh = lambda t: t.view(B, L, n, d).transpose(1, 2)
    i = torch.arange(L, dtype=torch.float64)
    dist = (i[:, None] - i[None, :]).abs()
    bias = -torch.tensor(slopes, dtype=torch.float64)[:, None, None] * dist
    keym = torch.from_numpy(mask.astype(bool))[:, None, None, :]
    bias = torch.where(keym, bias[None], torch.tensor(-math.inf, dtype=torch.float64))
    c = F.scaled_dot_product_attention(sh(q), sh(k), sh(v), attn_mask=bias)
    c = c.transpose(1, 2).reshape(B, L, H)
    y1 = F.layer_norm(F.linear(c, p["w_o"], p["b_o"]) + X, (H,), p["ln1_g"], p["ln1_b"], eps)
    u = F.linear(y1, p["w_1v"], p["b_1v"])
    a, g = u.chunk(2, dim=-1)
    z = F.gelu(a) * g
    return F.layer_norm(F.linear(z, p["w_2"], p["b_2"]) + y1, (H,), p["ln2_g"], p["ln2_b"], eps)


@pytest.mark.parametrize("case", ["tiny", "base_dims"])
def test_p14_torch_autograd_layer(case):
    import torch
    if case == "tiny":
        dims, lens, L = synth.TINY, [16, 9, 3, 1], 16
    else:
        dims, lens, L = synth.BASE, [128, 77], 128
    p = synth.make_layer_params(dims, 21, "stress")
    mask = synth.mask_from_lengths(np.array(lens), L)
    X = synth.make_hidden(mask, dims.hidden, 22)
    R = synth.make_grad(mask, dims.hidden, 23)
    slopes = O.alibi_slopes(dims.heads)
    Y, c = O.encoder_layer_forward(X, mask, slopes, p)
    dX, g = O.encoder_layer_backward(R, c)
    tp = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in p.items()}
    tX = torch.tensor(X, dtype=torch.float64, requires_grad=True)
    tY = _torch_layer(tX, mask, slopes, tp, 1e-12)
    m = torch.from_numpy(mask.astype(bool))
    (tY * torch.tensor(R, dtype=torch.float64) * m[..., None]).sum().backward()
    real = mask.astype(bool)
    assert np.max(np.abs(tY.detach().numpy()[real] - Y[real])) < 1e-10
    assert np.max(np.abs(tX.grad.numpy() * mask[..., None] - dX)) < 1e-10
    for k in p:
        ref = tp[k].grad.numpy()
        assert np.max(np.abs(ref - g[k])) < 1e-10 * max(1.0, np.abs(ref).max()), k


def test_p14_torch_autograd_head():
    import torch
    import torch.nn.functional as F
    dims = synth.TINY
    params = synth.make_model_params(dims, 5, "stress")
    batch = synth.make_batch("C1", 3)
    rng = np.random.default_rng(0)
    Y = rng.standard_normal((4, 16, dims.hidden))
    hp = {k: params[k] for k in synth.HEAD_KEYS}
    n = int((batch["labels"] != -100).sum())
    loss, dY, g, _ = O.mlm_head_forward_backward(Y, batch["labels"], batch["attention_mask"], hp, params["emb"], 1.0 / n)
    t = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in hp.items()}
    E = torch.tensor(params["emb"], dtype=torch.float64, requires_grad=True)
    tY = torch.tensor(Y, requires_grad=True)
    h = F.gelu(F.linear(tY, t["w_t"], t["b_t"]))
    u = F.layer_norm(h, (dims.hidden,), t["lnh_g"], t["lnh_b"], 1e-12)
    z = F.linear(u, E, t["b_dec"])
    tl = F.cross_entropy(z.view(-1, dims.vocab), torch.from_numpy(batch["labels"].astype(np.int64)).view(-1), ignore_index=-100)
    tl.backward()
    assert abs(tl.item() - loss) < 1e-12
    assert np.max(np.abs(tY.grad.numpy() - dY)) < 1e-12
    assert np.max(np.abs(E.grad.numpy() - g["emb"])) < 1e-12
    for k in hp:
        assert np.max(np.abs(t[k].grad.numpy() - g[k])) < 1e-12, k
