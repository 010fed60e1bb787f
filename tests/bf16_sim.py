"""Storage-precision model of the GPU step (TEST INFRASTRUCTURE: an error-budget tool, not the oracle).

The fp64 oracle (oracle/mosaicbert.py) is the parity reference.  This module re-runs the same
arithmetic in fp64 but rounds to bf16 (RNE) at a chosen set of *sites*: the places where the CUDA
path stores a tensor in bf16 (reading R25: bf16 storage, fp32 arithmetic; the
paper trains in bf16 mixed precision, with bf16 LayerNorm).  Comparing this model
with the exact oracle measures, before any GPU run, how far a bf16-storage implementation of the
step can be expected to sit from the exact result — the a-priori error bar of reading R33.

Sites (per encoder layer, forward):  x (layer input), qkv, p (attention probabilities fed to the
PV product), o, s1 (out-proj + residual), y1 (LN1 out), z (GeGLU out), gd (saved GeGLU factors),
s2 (down-proj + residual).  Backward: dy (layer output gradient), ds2, du, dy1, ds1, dc (attention
output gradient), ap (attention P and dS fed to the gradient products), dqkv.  Head: h_tp
(transform pre-activation), h_t, h_u, h_dz, h_du, h_dt (LN_h backward output after GeLU'), h_dh.
ALL = every site, i.e. the GPU path's storage."""
from __future__ import annotations

import math

import numpy as np
from scipy.special import erf

import oracle as O
import synth

FWD = ("x", "qkv", "p", "o", "s1", "y1", "z", "gd", "s2")
BWD = ("dy", "ds2", "du", "dy1", "ds1", "dc", "ap", "dqkv")
HEAD = ("h_tp", "h_t", "h_u", "h_dz", "h_du", "h_dt", "h_dh")
ALL = frozenset(FWD + BWD + HEAD)
BOUNDARY = frozenset(("x", "dy"))  # the R33 round-1 floor: only the tensors passed between layers


def _bf(a):
    return synth.bf16_round(np.asarray(a, dtype=np.float64)).astype(np.float64)


class _R:
    def __init__(self, sites, jitter=0.0, seed=0):
        self.sites = frozenset(sites)
        self.jitter = jitter  # relative perturbation before each rounding (fp32-accumulation noise model)
        self.rng = np.random.default_rng(seed)

    def __call__(self, site, a):
        a = np.asarray(a, dtype=np.float64)
        if site not in self.sites:
            return a
        if self.jitter:
            a = a * (1.0 + self.jitter * self.rng.standard_normal(a.shape))
        return _bf(a)


def _gelu(x):
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


def _gelu_grad(x):
    return 0.5 * (1.0 + erf(x / math.sqrt(2.0))) + x * np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)


def _attn_fwd(r, q, k, v, mask, slopes):
    B, L, n, d = q.shape
    lens = np.asarray(mask).sum(1)
    pos = np.arange(L)
    bias = -np.asarray(slopes)[:, None, None] * np.abs(pos[:, None] - pos[None, :])[None]
    s = np.einsum("bind,bjnd->bnij", q, k) / math.sqrt(d) + bias[None]
    keym = pos[None, :] < lens[:, None]  # [B, L]
    s = np.where(keym[:, None, None, :], s, -np.inf)
    mx = s.max(-1, keepdims=True)
    mx = np.where(np.isfinite(mx), mx, 0.0)
    e = np.exp(s - mx)
    l = e.sum(-1, keepdims=True)
    l = np.where(l > 0, l, 1.0)
    P = e / l
    # the kernels feed the unnormalised exponentials to the PV MMA in bf16 and divide by l after
    c = np.einsum("bnij,bjnd->bind", r("p", e), v) / np.transpose(l, (0, 2, 1, 3))
    return c, (q, k, v, P, lens)


def _attn_bwd(r, dC, cache):
    q, k, v, P, lens = cache
    d = q.shape[-1]
    Pb = r("ap", P)
    dv = np.einsum("bnij,bind->bjnd", Pb, dC)
    dp = np.einsum("bind,bjnd->bnij", dC, v)
    D = (P * dp).sum(-1, keepdims=True)
    ds = r("ap", P * (dp - D) / math.sqrt(d))
    dq = np.einsum("bnij,bjnd->bind", ds, k)
    dk = np.einsum("bnij,bind->bjnd", ds, q)
    return dq, dk, dv


def layer_forward(r, X, mask, slopes, p, eps, dropout=None):
    P = {k_: np.asarray(v_, dtype=np.float64) for k_, v_ in p.items()}
    B, L, H = X.shape
    n = len(slopes)
    D0, D1 = O.dropout_masks(mask, H, dropout)  # F2 (R32): the oracle's own masks
    X = r("x", X)
    QKV = r("qkv", X @ P["w_qkv"].T + P["b_qkv"])
    sp = lambda t: t.reshape(B, L, n, H // n)  # noqa: E731
    C4, ac = _attn_fwd(r, sp(QKV[..., :H]), sp(QKV[..., H:2 * H]), sp(QKV[..., 2 * H:]), mask, slopes)
    C = r("o", C4.reshape(B, L, H))
    S1 = r("s1", (C @ P["w_o"].T + P["b_o"]) * D0 + X)
    y1, ln1 = O.layer_norm(S1, P["ln1_g"], P["ln1_b"], eps)
    Y1 = r("y1", y1)
    U = Y1 @ P["w_1v"].T + P["b_1v"]
    I = U.shape[-1] // 2
    a, g = U[..., :I], U[..., I:]
    Z = r("z", _gelu(a) * g)
    Ga, Gg = r("gd", g * _gelu_grad(a)), r("gd", _gelu(a))
    S2 = r("s2", (Z @ P["w_2"].T + P["b_2"]) * D1 + Y1)
    Y, ln2 = O.layer_norm(S2, P["ln2_g"], P["ln2_b"], eps)
    return Y, dict(X=X, mask=np.asarray(mask), P=P, C=C, ac=ac, ln1=ln1, Y1=Y1, Z=Z, Ga=Ga, Gg=Gg, ln2=ln2, n=n,
                   D0=D0, D1=D1)


def layer_backward(r, dY, c):
    P, n = c["P"], c["n"]
    m = c["mask"][..., None].astype(np.float64)
    B, L, H = c["X"].shape
    fl = lambda t: t.reshape(-1, t.shape[-1])  # noqa: E731
    g = {}
    dY = r("dy", dY) * m
    dS2, g["ln2_g"], g["ln2_b"] = O.layer_norm_backward(dY, c["ln2"], P["ln2_g"])
    dS2f = dS2 * m
    dS2 = r("ds2", dS2f)
    # with F2 dropout the LN backward also writes the dropped-branch gradient; without, it is dS2
    dF = dS2 if np.isscalar(c["D1"]) else r("ds2", dS2f * c["D1"])
    g["w_2"] = fl(dF).T @ fl(c["Z"])
    g["b_2"] = fl(dF).sum(0)
    dZ = dF @ P["w_2"]
    dU = r("du", np.concatenate([dZ * c["Ga"], dZ * c["Gg"]], -1))
    g["w_1v"] = fl(dU).T @ fl(c["Y1"])
    g["b_1v"] = fl(dU).sum(0)
    dY1 = r("dy1", dU @ P["w_1v"] + dS2)
    dS1, g["ln1_g"], g["ln1_b"] = O.layer_norm_backward(dY1, c["ln1"], P["ln1_g"])
    dS1f = dS1 * m
    dS1 = r("ds1", dS1f)
    dA = dS1 if np.isscalar(c["D0"]) else r("ds1", dS1f * c["D0"])
    g["w_o"] = fl(dA).T @ fl(c["C"])
    g["b_o"] = fl(dA).sum(0)
    dC = r("dc", dA @ P["w_o"])
    dq, dk, dv = _attn_bwd(r, dC.reshape(B, L, n, H // n), c["ac"])
    dQKV = r("dqkv", np.concatenate([dq.reshape(B, L, H), dk.reshape(B, L, H), dv.reshape(B, L, H)], -1) * m)
    g["w_qkv"] = fl(dQKV).T @ fl(c["X"])
    g["b_qkv"] = fl(dQKV).sum(0)
    dX = (dQKV @ P["w_qkv"] + dS1) * m
    return dX, g


def head(r, Y, labels, mask, hp, emb, inv_norm, eps):
    lab = np.asarray(labels)
    sel = (lab != O.IGNORE) & (np.asarray(mask) != 0)
    bi = np.argwhere(sel)
    h = r("x", Y[bi[:, 0], bi[:, 1]])
    y = lab[bi[:, 0], bi[:, 1]]
    W_t, b_t, E = (np.asarray(hp[k], dtype=np.float64) for k in ("w_t", "b_t", "emb"))
    tp = r("h_tp", h @ W_t.T + b_t)
    t = r("h_t", _gelu(tp))
    u_, lnc = O.layer_norm(t, hp["lnh_g"], hp["lnh_b"], eps)
    u = r("h_u", u_)
    z = u @ E.T + np.asarray(hp["b_dec"], dtype=np.float64)
    mx = z.max(1, keepdims=True)
    lse = (mx + np.log(np.exp(z - mx).sum(1, keepdims=True)))[:, 0]
    rows = np.arange(len(y))
    loss = inv_norm * float(np.sum(lse - z[rows, y]))
    dz = np.exp(z - lse[:, None])
    dz[rows, y] -= 1.0
    dz = r("h_dz", dz * inv_norm)
    g = {"b_dec": dz.sum(0), "emb": dz.T @ u}
    du = r("h_du", dz @ E)
    dt, g["lnh_g"], g["lnh_b"] = O.layer_norm_backward(du, lnc, hp["lnh_g"])
    dtp = r("h_dt", dt * _gelu_grad(tp))
    g["w_t"] = dtp.T @ h
    g["b_t"] = dtp.sum(0)
    dY = np.zeros_like(Y)
    dY[bi[:, 0], bi[:, 1]] = r("h_dh", dtp @ W_t)
    return loss, dY, g, lse


def model_step(batch, params, heads, inv_norm, eps, sites=ALL, jitter=0.0, seed=0, dropout=None):
    """One micro-step (embedding -> layers -> MLM head+CE -> backward) with bf16 rounding at `sites`.
    dropout = dict(p, seed[, rows]) or None: layer li uses stream li (R32, as the oracle).
    Returns (loss, per-masked-row LSE, gradient at the embedding-LN output, gradients)."""
    r = _R(sites, jitter, seed)
    ids, mask, labels = batch["input_ids"], batch["attention_mask"], batch["labels"]
    slopes = O.alibi_slopes(heads)
    X, ec = O.embed_forward(ids, params["emb"], params["type_emb"], params["lne_g"], params["lne_b"], eps)
    caches = []
    for li, lp in enumerate(params["layers"]):
        X, c = layer_forward(r, X, mask, slopes, lp, eps, dict(dropout, stream=li) if dropout else None)
        caches.append(c)
    hp = {k: params[k] for k in ("w_t", "b_t", "lnh_g", "lnh_b", "b_dec", "emb")}
    loss, dY, g, lse = head(r, X, labels, mask, hp, params["emb"], inv_norm, eps)
    g["layers"] = [None] * len(caches)
    for li in range(len(caches) - 1, -1, -1):
        dY, g["layers"][li] = layer_backward(r, dY, caches[li])
    dY = r("dy", dY)
    dE, g["type_emb"], g["lne_g"], g["lne_b"] = O.embed_backward(dY, ids, mask, ec, params["lne_g"],
                                                                 params["emb"].shape[0])
    g["emb"] = g["emb"] + dE
    return loss, lse, dY, g
