"""fp64 oracle: MosaicBERT encoder layer / embedding / MLM head, forward and backward, on the
PADDED batch.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Notation follows the paper: q_i, K, m (Eq. 1), x, W1, V, W2 (Eq. 2).
All arrays are numpy float64; inputs arrive as float32 bf16-exact values and are upcast exactly.
"""
from __future__ import annotations

import math
import numpy as np
from scipy.special import erf

from .philox import dropout_keep, dropout_scale

__all__ = [
    "MB_OK", "MB_ERR_MASK_LAYOUT", "IGNORE",
    "alibi_slopes", "alibi_bias", "unpad_index", "unpad", "pad",
    "gelu", "gelu_grad", "layer_norm", "layer_norm_backward", "softmax",
    "attention_forward", "attention_backward",
    "encoder_layer_forward", "encoder_layer_backward",
    "embed_forward", "embed_backward", "mlm_head_forward_backward",
    "model_forward_backward", "param_count", "mfu", "dropout_masks",
]

MB_OK = 0
MB_ERR_MASK_LAYOUT = 4
IGNORE = -100


def f64(x):
    return np.asarray(x, dtype=np.float64)


# ---------------------------------------------------------------------------------------------
# ALiBi (Eq. 1)
# ---------------------------------------------------------------------------------------------
def alibi_slopes(n_heads: int) -> np.ndarray:
    """m_h = 2^(-8(h+1)/n), h = 0..n-1: "a geometric sequence ... each head has a ratio of
    2^{-8/n}" (reading R3/R27: first term = ratio).  Returned in float64."""
    if n_heads <= 0:
        raise ValueError("heads must be positive (S:126)")
    return np.array([2.0 ** (-8.0 * (h + 1) / n_heads) for h in range(n_heads)], dtype=np.float64)


def alibi_bias(L: int, m: float) -> np.ndarray:
    """-m * abs(i - j) for i, j in [0, L): the bias matrix of Eq. 1 (reading R4)."""
    i = np.arange(L)
    return -float(m) * np.abs(i[:, None] - i[None, :]).astype(np.float64)


# ---------------------------------------------------------------------------------------------
# Unpadding (SPEC unpad S:336-361)
# ---------------------------------------------------------------------------------------------
def unpad_index(mask):
    """Brute-force unpad index.
    seqlen[b] = sum_l mask[b,l]; cu_seqlens = [0, cumsum]; indices = ascending flat positions
    b*L+l where mask==1; max_seqlen = max seqlen; status = MASK_LAYOUT if some row is not a
    prefix of ones (right padding, reading R6), else OK."""
    mask = np.asarray(mask)
    B, L = mask.shape
    seqlen = mask.astype(np.int64).sum(axis=1)
    cu = np.concatenate([[0], np.cumsum(seqlen)]).astype(np.int32)
    indices = np.flatnonzero(mask.reshape(-1)).astype(np.int32)
    max_seqlen = int(seqlen.max()) if B > 0 else 0
    status = MB_OK
    for b in range(B):
        if not mask[b, : seqlen[b]].all():
            status = MB_ERR_MASK_LAYOUT
    return cu, indices, max_seqlen, status


def unpad(x, indices):
    """packed[t] = x.reshape(B*L, ...)[indices[t]]  ("concatenate all the examples")."""
    x = np.asarray(x)
    return x.reshape((-1,) + x.shape[2:])[indices]


def pad(packed, indices, B, L):
    """Inverse of unpad: real rows restored, all other rows exactly 0."""
    packed = np.asarray(packed)
    out = np.zeros((B * L,) + packed.shape[1:], dtype=packed.dtype)
    out[indices] = packed
    return out.reshape((B, L) + packed.shape[1:])


# ---------------------------------------------------------------------------------------------
# elementwise pieces
# ---------------------------------------------------------------------------------------------
def gelu(x):
    """GeLU(x) = x * Phi(x), exact erf form (P:136 footnote; reading R7)."""
    x = f64(x)
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


def gelu_grad(x):
    """d/dx [x Phi(x)] = Phi(x) + x phi(x)."""
    x = f64(x)
    cdf = 0.5 * (1.0 + erf(x / math.sqrt(2.0)))
    pdf = np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)
    return cdf + x * pdf


def softmax(s, axis=-1):
    """Max-subtracted softmax; -inf entries map to exactly 0."""
    s = f64(s)
    mx = np.max(s, axis=axis, keepdims=True)
    e = np.exp(s - mx)
    return e / e.sum(axis=axis, keepdims=True)


def layer_norm(v, g, b, eps):
    """LN(v) = (v - mu)/sqrt(sigma^2 + eps) * gamma + beta, biased variance (
    readings R11/R12).  Returns y and the cache (xhat, rstd)."""
    v = f64(v)
    mu = v.mean(axis=-1, keepdims=True)
    var = ((v - mu) ** 2).mean(axis=-1, keepdims=True)
    r = 1.0 / np.sqrt(var + eps)
    xhat = (v - mu) * r
    return xhat * f64(g) + f64(b), (xhat, r)


def layer_norm_backward(dy, cache, g):
    """dv = r (gdy - mean(gdy) - xhat mean(gdy xhat)), gdy = dy*gamma; dgamma = sum dy xhat,
    dbeta = sum dy (sums over every leading axis)."""
    xhat, r = cache
    dy = f64(dy)
    gdy = dy * f64(g)
    dv = r * (gdy - gdy.mean(axis=-1, keepdims=True)
              - xhat * (gdy * xhat).mean(axis=-1, keepdims=True))
    H = dy.shape[-1]
    dg = (dy * xhat).reshape(-1, H).sum(axis=0)
    db = dy.reshape(-1, H).sum(axis=0)
    return dv, dg, db


# ---------------------------------------------------------------------------------------------
# ALiBi attention on the padded batch (Eq. 1)
# ---------------------------------------------------------------------------------------------
def attention_forward(q, k, v, mask, slopes):
    """q, k, v: [B, L, n, d]; mask [B, L]; slopes [n].
    s_ij = q_i . k_j / sqrt(d) - m_h |i - j| for keys j < l_b, -inf for pad keys (Eq. 1 P:127;
    readings R2 scale-then-bias, R4 symmetric distance, R5 pad keys excluded).
    P = softmax_j(s); C_i = sum_j P_ij v_j; LSE_i = log sum_j exp(s_ij).
    Rows of zero-length sequences are skipped (output 0, R5).  No dropout (R14)."""
    q, k, v = f64(q), f64(k), f64(v)
    B, L, n, d = q.shape
    slopes = f64(slopes)
    lens = np.asarray(mask).sum(axis=1)
    C = np.zeros_like(q)
    P = np.zeros((B, n, L, L))
    LSE = np.zeros((B, n, L))
    for b in range(B):
        lb = int(lens[b])
        if lb == 0:
            continue
        for h in range(n):
            s = q[b, :, h, :] @ k[b, :, h, :].T / math.sqrt(d) + alibi_bias(L, slopes[h])
            s[:, lb:] = -np.inf
            mx = s.max(axis=1, keepdims=True)
            e = np.exp(s - mx)
            z = e.sum(axis=1, keepdims=True)
            p = e / z
            P[b, h] = p
            LSE[b, h] = (mx + np.log(z))[:, 0]
            C[b, :, h, :] = p @ v[b, :, h, :]
    return C, (q, k, v, P, lens)


def attention_backward(dC, cache):
    """dV = P^T dC, dP = dC V^T, dS = P (dP - rowsum(dP P)), dQ = dS K / sqrt d, dK = dS^T Q / sqrt d.
    Slopes are constants and receive no gradient."""
    q, k, v, P, lens = cache
    dC = f64(dC)
    B, L, n, d = q.shape
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    for b in range(B):
        if int(lens[b]) == 0:
            continue
        for h in range(n):
            p = P[b, h]
            dc = dC[b, :, h, :]
            dv[b, :, h, :] = p.T @ dc
            dp = dc @ v[b, :, h, :].T
            ds = p * (dp - (dp * p).sum(axis=1, keepdims=True))
            dq[b, :, h, :] = ds @ k[b, :, h, :] / math.sqrt(d)
            dk[b, :, h, :] = ds.T @ q[b, :, h, :] / math.sqrt(d)
    return dq, dk, dv


# ---------------------------------------------------------------------------------------------
# one post-LN encoder layer (readings R1, R8-R10)
# ---------------------------------------------------------------------------------------------
def _split_heads(x, n):
    B, L, H = x.shape
    return x.reshape(B, L, n, H // n)


def dropout_masks(mask, H, dropout):
    """Padded [B, L, H] keep/P(keep) multipliers of the two F2 dropout sites (R32) for one layer:
    the packed row of real position (b, l) is its rank in row-major order (P:147 packing), pad
    positions get 0.  dropout = dict(p, seed, stream) (stream = layer index) or None -> (1, 1);
    an optional dropout["rows"] gives the packed row of each real position (row-major order) when
    the batch is a subset of a larger packed micro-batch."""
    if not dropout or dropout.get("p", 0.0) == 0.0:
        return 1.0, 1.0
    mk = np.asarray(mask).astype(bool)
    T = int(mk.sum())
    out = []
    for site in (0, 1):
        keep = dropout_keep(T, H, dropout["p"], dropout["seed"], dropout["stream"], site, dropout.get("rows"))
        d = np.zeros(mk.shape + (H,))
        d[mk] = keep * dropout_scale(dropout["p"])
        out.append(d)
    return out[0], out[1]


def encoder_layer_forward(X, mask, slopes, p, eps=1e-12, dropout=None):
    """X [B, L, H] padded; p = dict of W[out,in] / bias / LN params (float arrays).
      QKV = X W_qkv^T + b_qkv, columns (3, heads, d)                       (R9)
      C = ALiBi attention (Eq. 1); A = C W_o^T + b_o
      Y1 = LN(drop_0(A) + X; gamma1, beta1)                                 (post-LN, R1)
      U = Y1 W_1v^T + b_1v; a = U[:, :I] (W1 half), g = U[:, I:] (V half)   (fused GLU P:685, R8)
      Z = GeLU(a) * g; F = Z W_2^T + b_2                                   (Eq. 2)
      Y = LN(drop_1(F) + Y1; gamma2, beta2)
    drop_s = the F2 dropout of site s ("0.1 dropout to the feedforward layers"; placement
    after each output projection, before the residual: SURVEY §8f F2, R32); identity when
    dropout is None or p = 0 (R13).  Returns Y and a cache for the backward."""
    X = f64(X)
    B, L, H = X.shape
    D0, D1 = dropout_masks(mask, H, dropout)
    n = len(slopes)
    P = {k_: f64(v_) for k_, v_ in p.items()}
    QKV = X @ P["w_qkv"].T + P["b_qkv"]
    Q, K, V = QKV[..., :H], QKV[..., H:2 * H], QKV[..., 2 * H:]
    C4, acache = attention_forward(_split_heads(Q, n), _split_heads(K, n), _split_heads(V, n),
                                   mask, slopes)
    C = C4.reshape(B, L, H)
    A = C @ P["w_o"].T + P["b_o"]
    S1 = A * D0 + X
    Y1, ln1 = layer_norm(S1, P["ln1_g"], P["ln1_b"], eps)
    U = Y1 @ P["w_1v"].T + P["b_1v"]
    I = U.shape[-1] // 2
    a, g = U[..., :I], U[..., I:]
    Z = gelu(a) * g
    F = Z @ P["w_2"].T + P["b_2"]
    S2 = F * D1 + Y1
    Y, ln2 = layer_norm(S2, P["ln2_g"], P["ln2_b"], eps)
    cache = dict(X=X, mask=np.asarray(mask), n=n, P=P, QKV=QKV, C=C, acache=acache, S1=S1,
                 ln1=ln1, Y1=Y1, U=U, Z=Z, S2=S2, ln2=ln2, D0=D0, D1=D1)
    return Y, cache


def encoder_layer_backward(dY, cache):
    """Analytic backward of encoder_layer_forward (SURVEY §8c.1 rules).  Upstream gradients at
    pad rows are zeroed (pad rows contribute nothing, pin P9).  Returns dX and the parameter
    gradients (same keys as the params)."""
    P = cache["P"]
    m = cache["mask"][..., None].astype(np.float64)
    dY = f64(dY) * m
    X, n = cache["X"], cache["n"]
    B, L, H = X.shape
    I = cache["U"].shape[-1] // 2
    flat = lambda t: t.reshape(-1, t.shape[-1])
    g_ = {}
    # Y = LN2(S2)
    dS2, g_["ln2_g"], g_["ln2_b"] = layer_norm_backward(dY, cache["ln2"], P["ln2_g"])
    dS2 = dS2 * m
    # S2 = drop_1(F) + Y1, F = Z W2^T + b2
    dF = dS2 * cache["D1"]
    g_["w_2"] = flat(dF).T @ flat(cache["Z"])
    g_["b_2"] = flat(dF).sum(axis=0)
    dZ = dF @ P["w_2"]
    U = cache["U"]
    a, g = U[..., :I], U[..., I:]
    da = dZ * g * gelu_grad(a)
    dg = dZ * gelu(a)
    dU = np.concatenate([da, dg], axis=-1)
    g_["w_1v"] = flat(dU).T @ flat(cache["Y1"])
    g_["b_1v"] = flat(dU).sum(axis=0)
    dY1 = dU @ P["w_1v"] + dS2
    # Y1 = LN1(S1)
    dS1, g_["ln1_g"], g_["ln1_b"] = layer_norm_backward(dY1, cache["ln1"], P["ln1_g"])
    dS1 = dS1 * m
    # S1 = drop_0(A) + X, A = C Wo^T + bo
    dA = dS1 * cache["D0"]
    g_["w_o"] = flat(dA).T @ flat(cache["C"])
    g_["b_o"] = flat(dA).sum(axis=0)
    dC = dA @ P["w_o"]
    dq, dk, dv = attention_backward(_split_heads(dC, n), cache["acache"])
    dQKV = np.concatenate([dq.reshape(B, L, H), dk.reshape(B, L, H), dv.reshape(B, L, H)], axis=-1)
    dQKV = dQKV * m
    g_["w_qkv"] = flat(dQKV).T @ flat(X)
    g_["b_qkv"] = flat(dQKV).sum(axis=0)
    dX = (dQKV @ P["w_qkv"] + dS1) * m
    return dX, g_


# ---------------------------------------------------------------------------------------------
# embedding (no position table; BERT token + type embedding + LN, readings R16/R17/R28)
# ---------------------------------------------------------------------------------------------
def embed_forward(ids, emb, type_emb, g, b, eps=1e-12):
    """X0 = LN_e(E_tok[id] + E_type[0]) at every position (pad rows included; they are ignored)."""
    v = f64(emb)[np.asarray(ids)] + f64(type_emb)[0]
    y, c = layer_norm(v, g, b, eps)
    return y, c


def embed_backward(dX0, ids, mask, cache, g, V):
    """dE_tok[id] += dx (real rows only), dE_type[0] += sum dx, dgamma_e, dbeta_e."""
    m = np.asarray(mask)[..., None].astype(np.float64)
    dX0 = f64(dX0) * m
    dv, dg, db = layer_norm_backward(dX0, cache, g)
    dv = dv * m
    H = dv.shape[-1]
    dE = np.zeros((V, H))
    np.add.at(dE, np.asarray(ids).reshape(-1), dv.reshape(-1, H))
    dT = np.zeros((2, H))
    dT[0] = dv.reshape(-1, H).sum(axis=0)
    return dE, dT, dg, db


# ---------------------------------------------------------------------------------------------
# MLM head on masked tokens + softmax cross-entropy (R15, R18)
# ---------------------------------------------------------------------------------------------
def mlm_head_forward_backward(Y, labels, mask, hp, emb, inv_norm, eps=1e-12):
    """For every real position (b, i) with label y != -100:
        t = GeLU(Y[b,i] W_t^T + b_t); u = LN_h(t); z = u E_tok^T + b_dec  (decoder tied to E_tok)
        loss = inv_norm * sum (logsumexp(z) - z_y)
    inv_norm = 1 / (global number of labelled positions) (R18).  Returns loss, dY, grads
    (w_t, b_t, lnh_g, lnh_b, b_dec, emb) and per-row LSE."""
    Y = f64(Y)
    B, L, H = Y.shape
    lab = np.asarray(labels)
    sel = (lab != IGNORE) & (np.asarray(mask) != 0)
    bi = np.argwhere(sel)
    h = Y[bi[:, 0], bi[:, 1]]
    y = lab[bi[:, 0], bi[:, 1]]
    W_t, b_t = f64(hp["w_t"]), f64(hp["b_t"])
    E = f64(emb)
    tp = h @ W_t.T + b_t
    t = gelu(tp)
    u, lnc = layer_norm(t, hp["lnh_g"], hp["lnh_b"], eps)
    z = u @ E.T + f64(hp["b_dec"])
    mx = z.max(axis=1, keepdims=True)
    lse = (mx + np.log(np.exp(z - mx).sum(axis=1, keepdims=True)))[:, 0]
    rows = np.arange(len(y))
    loss = inv_norm * float(np.sum(lse - z[rows, y]))
    dz = np.exp(z - lse[:, None])
    dz[rows, y] -= 1.0
    dz *= inv_norm
    g_ = {"b_dec": dz.sum(axis=0), "emb": dz.T @ u}
    du = dz @ E
    dt, g_["lnh_g"], g_["lnh_b"] = layer_norm_backward(du, lnc, hp["lnh_g"])
    dtp = dt * gelu_grad(tp)
    g_["w_t"] = dtp.T @ h
    g_["b_t"] = dtp.sum(axis=0)
    dh = dtp @ W_t
    dY = np.zeros_like(Y)
    dY[bi[:, 0], bi[:, 1]] = dh
    return loss, dY, g_, lse


# ---------------------------------------------------------------------------------------------
# the whole step: embedding -> layers -> MLM head+CE -> backward
# ---------------------------------------------------------------------------------------------
def model_forward_backward(batch, params, slopes, eps=1e-12, inv_norm=None, dropout=None):
    """One micro-step of MosaicBERT pretraining on the padded batch (SURVEY §3 call stack 1).
    dropout = dict(p, seed) or None: layer li uses stream li (R32).
    Returns loss and gradients for every parameter (tied E_tok receives decoder + embedding)."""
    ids, mask, labels = batch["input_ids"], batch["attention_mask"], batch["labels"]
    V = params["emb"].shape[0]
    n_lab = int(((np.asarray(labels) != IGNORE) & (np.asarray(mask) != 0)).sum())
    if inv_norm is None:
        inv_norm = 1.0 / max(n_lab, 1)
    X, ecache = embed_forward(ids, params["emb"], params["type_emb"], params["lne_g"],
                              params["lne_b"], eps)
    caches = []
    for li, lp in enumerate(params["layers"]):
        dli = dict(dropout, stream=li) if dropout else None
        X, c = encoder_layer_forward(X, mask, slopes, lp, eps, dli)
        caches.append(c)
    hp = {k: params[k] for k in ("w_t", "b_t", "lnh_g", "lnh_b", "b_dec")}
    loss, dY, hg, _ = mlm_head_forward_backward(X, labels, mask, hp, params["emb"], inv_norm, eps)
    grads = {"layers": [None] * len(caches)}
    for li in range(len(caches) - 1, -1, -1):
        dY, grads["layers"][li] = encoder_layer_backward(dY, caches[li])
    dE, dT, dg, db = embed_backward(dY, ids, mask, ecache, params["lne_g"], V)
    grads.update(hg)
    grads["emb"] = grads["emb"] + dE
    grads["type_emb"], grads["lne_g"], grads["lne_b"] = dT, dg, db
    return loss, grads


# ---------------------------------------------------------------------------------------------
# accounting (Eq. 3; parameter counts P:141)
# ---------------------------------------------------------------------------------------------
def param_count(hidden, heads, intermediate, vocab, layers, glu=True, position_rows=0,
                type_rows=2, tied_decoder=True):
    """Learnable scalars of the architecture of SURVEY §8c (readings R10, R15-R17)."""
    H, I = hidden, intermediate
    emb = vocab * H + type_rows * H + position_rows * H + 2 * H
    attn = 3 * H * H + 3 * H + H * H + H + 2 * H
    ffn = (2 if glu else 1) * (I * H + I) + I * H + H + 2 * H
    head = H * H + H + 2 * H + vocab + (0 if tied_decoder else vocab * H)
    return emb + layers * (attn + ffn) + head


def mfu(tokens_per_s, n_params, n_gpus, peak_flops):
    """MFU = 6 N T_obs / (n_gpus T_theoretical)  (Eq. 3)."""
    return 6.0 * n_params * tokens_per_s / (n_gpus * peak_flops)
