"""GPU parity of every kernel behind the C ABI against the fp64 oracle (or, for the plain GEMM, the
fp64 product of the same bf16 operands).  Integer work is compared bit-exactly."""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from parity import check, np64, to_dev

pytestmark = pytest.mark.gpu

mb = pytest.importorskip("paper_2312_17482_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mb.lib()


BF = torch.bfloat16
I32 = torch.int32


def _bf(a):
    return to_dev(a, torch.float32).to(BF)


# ------------------------------------------------------------------------------------ A1 / A2
MASK_CASES = {
    "C1": lambda: synth.make_batch("C1", 0)["attention_mask"],
    "C2": lambda: synth.make_batch("C2", 2000)["attention_mask"],
    "C5": lambda: synth.make_batch("C5", 5000)["attention_mask"],
    "C4": lambda: synth.make_batch("C4", 4000)["attention_mask"],
    "zero_rows": lambda: synth.mask_from_lengths(np.array([0, 5, 0, 3, 0]), 7),
    "L1": lambda: synth.mask_from_lengths(np.array([1, 0, 1, 1]), 1),
    "big_ragged": lambda: synth.mask_from_lengths(np.random.default_rng(0).integers(0, 301, 3000), 300),
    "all_zero": lambda: np.zeros((4, 9), dtype=np.int32),
    "many_rows": lambda: synth.mask_from_lengths(np.random.default_rng(1).integers(0, 65, 20000), 64),
}


@pytest.mark.parametrize("case", sorted(MASK_CASES))
def test_unpad_index_bitexact(case):
    mask = MASK_CASES[case]().astype(np.int32)
    cu, idx, meta = mb.unpad_index(to_dev(mask, I32))
    torch.cuda.synchronize()
    ocu, oidx, omax, ost = O.unpad_index(mask)
    m = meta.cpu().numpy()
    assert m[0] == len(oidx) and m[1] == omax and m[2] == ost
    assert np.array_equal(cu.cpu().numpy(), ocu)
    assert np.array_equal(idx.cpu().numpy()[: m[0]], oidx)


def test_unpad_index_nonprefix_status():
    mask = np.array([[1, 0, 1, 0], [1, 1, 0, 0]], dtype=np.int32)
    _, idx, meta = mb.unpad_index(to_dev(mask, I32))
    m = meta.cpu().numpy()
    assert m[2] == O.MB_ERR_MASK_LAYOUT
    assert idx.cpu().numpy()[: m[0]].tolist() == O.unpad_index(mask)[1].tolist()


@pytest.mark.parametrize("cfg", ["C1", "C5"])
def test_mlm_select_bitexact(cfg):
    bt = synth.make_batch(cfg, 7)
    mask, labels = bt["attention_mask"], bt["labels"]
    V = synth.CONFIGS[cfg].dims.vocab
    cu, idx, meta = mb.unpad_index(to_dev(mask, I32))
    rows, labs = mb.mlm_select(to_dev(labels, I32).reshape(-1), idx, V, meta)
    m = meta.cpu().numpy()
    _, oidx, _, _ = O.unpad_index(mask)
    lab_packed = labels.reshape(-1)[oidx]
    want = np.flatnonzero(lab_packed != -100)
    assert m[3] == len(want) and m[2] == 0
    assert np.array_equal(rows.cpu().numpy()[: m[3]], want)
    assert np.array_equal(labs.cpu().numpy()[: m[3]], lab_packed[want])


def test_mlm_select_label_range():
    mask = np.ones((1, 4), dtype=np.int32)
    labels = np.array([[-100, 5, 200, -100]], dtype=np.int32)
    cu, idx, meta = mb.unpad_index(to_dev(mask, I32))
    mb.mlm_select(to_dev(labels, I32).reshape(-1), idx, 128, meta)
    assert meta.cpu().numpy()[2] == 5  # MB_ERR_LABEL_RANGE


@pytest.mark.parametrize("H", [64, 768])
def test_gather_scatter_roundtrip_bitwise(H):
    mask = synth.make_batch("C5", 3, B=64)["attention_mask"]
    B, L = mask.shape
    x = synth.make_hidden(mask, H, 1)
    xd = _bf(x.reshape(B * L, H))
    cu, idx, meta = mb.unpad_index(to_dev(mask, I32))
    nnz = int(meta[0].item())
    packed = torch.empty(nnz, H, dtype=BF, device="cuda")
    mb.gather_rows(xd, idx, nnz, packed)
    _, oidx, _, _ = O.unpad_index(mask)
    assert torch.equal(packed.cpu(), xd.cpu()[torch.from_numpy(oidx).long()])
    back = torch.full((B * L, H), 7.0, dtype=BF, device="cuda")
    mb.scatter_rows(packed, idx, nnz, B * L, back)
    want = torch.from_numpy(O.pad(O.unpad(x, oidx), oidx, B, L).reshape(B * L, H)).to(BF)
    assert torch.equal(back.cpu(), want)


# ------------------------------------------------------------------------------------ A7 LayerNorm
@pytest.mark.parametrize("H", [64, 768, 1024])
@pytest.mark.parametrize("gelu", [False, True])
def test_layernorm_fwd_bwd(H, gelu):
    rng = np.random.default_rng(H)
    n = 333
    x = synth.bf16_round(rng.standard_normal((n, H)) * 3 + 1)
    g = synth.bf16_round(1 + 0.1 * rng.standard_normal(H))
    b = synth.bf16_round(0.1 * rng.standard_normal(H))
    dy = synth.bf16_round(rng.standard_normal((n, H)))
    pre = synth.bf16_round(rng.standard_normal((n, H)))
    y = torch.empty(n, H, dtype=BF, device="cuda")
    st = torch.empty(n, 2, dtype=torch.float32, device="cuda")
    mb.layernorm_forward(_bf(x), _bf(g), _bf(b), 1e-12, y, st)
    yo, cache = O.layer_norm(x, g, b, 1e-12)
    check("ln.y", np64(y), yo, max_rel=1e-2)
    xhat, r = cache
    check("ln.rstd", np64(st)[:, 1], r[:, 0], max_rel=1e-5)
    dx = torch.empty(n, H, dtype=BF, device="cuda")
    dg = torch.zeros(H, device="cuda")
    dbb = torch.zeros(H, device="cuda")
    ds = torch.zeros(H, device="cuda")
    mb.layernorm_backward(_bf(dy), _bf(x), st, _bf(g), dx, dg, dbb, ds, gelu_pre=_bf(pre) if gelu else None)
    dxo, dgo, dbo = O.layer_norm_backward(dy, cache, g)
    if gelu:
        dxo = dxo * O.gelu_grad(pre)
    check("ln.dx", np64(dx), dxo)
    check("ln.dgamma", np64(dg), dgo)
    check("ln.dbeta", np64(dbb), dbo, max_rel=1e-4)
    check("ln.dsum", np64(ds), dxo.sum(0))


# ------------------------------------------------------------------------------------ GEMM
GEMM_SHAPES = [(296, 200, 136), (1000, 768, 768), (136, 64, 64), (264, 512, 1000), (8, 8, 8)]  # M, N % 8 == 0 (TMA strides)


@pytest.mark.parametrize("shape", GEMM_SHAPES)
@pytest.mark.parametrize("a_t,b_t", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_gemm_transposes_bf16(shape, a_t, b_t):
    M, N, K = shape
    rng = np.random.default_rng(M + N + K + 10 * a_t + b_t)
    A = synth.bf16_round(rng.standard_normal((K, M) if a_t else (M, K)))
    Bm = synth.bf16_round(rng.standard_normal((K, N) if b_t else (N, K)))
    bias = synth.bf16_round(rng.standard_normal(N))
    res = synth.bf16_round(rng.standard_normal((M, N)))
    ref = (A.T if a_t else A).astype(np.float64) @ (Bm if b_t else Bm.T).astype(np.float64) + bias + res
    C = torch.empty(M, N, dtype=BF, device="cuda")
    mb.gemm(M, N, K, _bf(A), M if a_t else K, a_t, _bf(Bm), N if b_t else K, b_t, C, N, 0, bias=_bf(bias),
            residual=_bf(res), ldr=N)
    check(f"gemm{shape}{a_t}{b_t}", np64(C), ref, max_rel=1e-2, min_cos=0.9999)


@pytest.mark.parametrize("shape", [(768, 768, 4096), (2304, 768, 333), (64, 64, 40)])
def test_gemm_f32_acc_weight_grad(shape):
    """dW += dY^T X (both operands MN-major, split-K, fp32 atomics into an existing buffer)."""
    M, N, K = shape
    rng = np.random.default_rng(K)
    dY = synth.bf16_round(rng.standard_normal((K, M)))
    X = synth.bf16_round(rng.standard_normal((K, N)))
    C0 = rng.standard_normal((M, N)).astype(np.float32)
    Cd = to_dev(C0, torch.float32)
    mb.gemm(M, N, K, _bf(dY), M, 1, _bf(X), N, 1, Cd, N, 1)
    ref = C0 + dY.T.astype(np.float64) @ X.astype(np.float64)
    check("gemm.f32acc", np64(Cd), ref, max_rel=1e-4, min_cos=0.999999)


@pytest.mark.parametrize("shape", [(768, 768, 4096), (6144, 768, 1000), (128, 64, 40), (30528, 768, 300)])
def test_gemm_wgrad_fused_bias_grad(shape):
    """dW += dY^T X and db += column sums of dY (tensor-core all-ones MMA), split-K into fp32."""
    M, N, K = shape
    rng = np.random.default_rng(M + K)
    dY = synth.bf16_round(rng.standard_normal((K, M)))
    X = synth.bf16_round(rng.standard_normal((K, N)))
    W0 = rng.standard_normal((M, N)).astype(np.float32)
    b0 = rng.standard_normal(M).astype(np.float32)
    Wd, bd = to_dev(W0, torch.float32), to_dev(b0, torch.float32)
    mb._lib.gemm_wgrad(M, N, K, _bf(dY), M, _bf(X), N, Wd, N, bd)
    check("wgrad.dW", np64(Wd), W0 + dY.T.astype(np.float64) @ X.astype(np.float64), max_rel=1e-4, min_cos=0.999999)
    check("wgrad.db", np64(bd), b0 + dY.astype(np.float64).sum(0), max_rel=1e-4, min_cos=0.999999)


def test_gemm_f32_and_gelu_aux():
    M, N, K = 200, 256, 192
    rng = np.random.default_rng(1)
    A = synth.bf16_round(rng.standard_normal((M, K)))
    W = synth.bf16_round(rng.standard_normal((N, K)) / np.sqrt(K))
    b = synth.bf16_round(rng.standard_normal(N))
    ref = A.astype(np.float64) @ W.T.astype(np.float64) + b
    C = torch.empty(M, N, dtype=torch.float32, device="cuda")
    mb.gemm(M, N, K, _bf(A), K, 0, _bf(W), K, 0, C, N, 2, bias=_bf(b))
    check("gemm.f32", np64(C), ref, max_rel=1e-4, min_cos=0.999999)
    G = torch.empty(M, N, dtype=BF, device="cuda")
    pre = torch.empty(M, N, dtype=BF, device="cuda")
    mb.gemm(M, N, K, _bf(A), K, 0, _bf(W), K, 0, G, N, 3, bias=_bf(b), aux=pre, ldaux=N)
    check("gemm.pre", np64(pre), ref, max_rel=1e-2)
    check("gemm.gelu", np64(G), O.gelu(ref), max_rel=1e-2)


# ------------------------------------------------------------------------------------ GeGLU
@pytest.mark.parametrize("H,I", [(64, 256), (768, 3072)])
def test_geglu_fwd_bwd(H, I):
    n = 300
    rng = np.random.default_rng(H)
    X = synth.bf16_round(rng.standard_normal((n, H)))
    W = synth.bf16_round(rng.standard_normal((2 * I, H)) / np.sqrt(H))
    b = synth.bf16_round(0.1 * rng.standard_normal(2 * I))
    W2 = synth.bf16_round(rng.standard_normal((H, I)) / np.sqrt(I))
    dF = synth.bf16_round(rng.standard_normal((n, H)))
    Gd = torch.empty(n, 2 * I, dtype=BF, device="cuda")
    Z = torch.empty(n, I, dtype=BF, device="cuda")
    mb.geglu_forward(_bf(X), _bf(W), _bf(b), Gd, Z)
    Uo = X.astype(np.float64) @ W.T.astype(np.float64) + b
    a, g = Uo[:, :I], Uo[:, I:]
    check("geglu.Z", np64(Z), O.gelu(a) * g, max_rel=1e-2)
    check("geglu.Gd_a", np64(Gd)[:, :I], g * O.gelu_grad(a), max_rel=1e-2)
    check("geglu.Gd_g", np64(Gd)[:, I:], O.gelu(a), max_rel=1e-2)
    dU = torch.empty(n, 2 * I, dtype=BF, device="cuda")
    mb.geglu_backward(_bf(dF), _bf(W2), Gd, dU)
    dZ = dF.astype(np.float64) @ W2.astype(np.float64)
    check("geglu.da", np64(dU)[:, :I], dZ * g * O.gelu_grad(a))
    check("geglu.dg", np64(dU)[:, I:], dZ * O.gelu(a))


# ------------------------------------------------------------------------------------ attention
ATTN_CASES = {
    "tiny_d32": (2, 32, [16, 9, 3, 1]),
    "base_d64_ragged": (12, 64, [128, 77, 1, 64, 100, 2]),
    "full128": (12, 64, [128] * 6),
    "multi_tile_512": (4, 64, [512, 300, 129, 128, 1]),
    "d32_multi": (2, 32, [200, 17]),
    "long_1024": (2, 64, [1024, 700, 5, 129]),   # F4
    "long_2048_d32": (1, 32, [2048, 1100]),      # F4
}


def _attn_inputs(heads, d, lens, seed):
    rng = np.random.default_rng(seed)
    H = heads * d
    lens = np.array(lens)
    Lmax = int(lens.max())
    mask = synth.mask_from_lengths(lens, Lmax)
    qkv_p = synth.bf16_round(rng.standard_normal((len(lens), Lmax, 3 * H)) * 1.5)
    do_p = synth.bf16_round(rng.standard_normal((len(lens), Lmax, H))) * mask[..., None]
    return mask, qkv_p, do_p


@pytest.mark.parametrize("case", sorted(ATTN_CASES))
def test_attention_fwd_bwd(case):
    heads, d, lens = ATTN_CASES[case]
    H = heads * d
    mask, qkv_p, do_p = _attn_inputs(heads, d, lens, len(case))
    B, Lmax = mask.shape
    cu, oidx, maxlen, _ = O.unpad_index(mask)
    nnz = len(oidx)
    slopes_np = mb.alibi_slopes(heads)
    qkv = _bf(O.unpad(qkv_p, oidx))
    dO = _bf(O.unpad(do_p, oidx))
    cud = to_dev(cu, I32)
    sl = to_dev(slopes_np, torch.float32)
    Od = torch.empty(nnz, H, dtype=BF, device="cuda")
    lse = torch.empty(heads, nnz, dtype=torch.float32, device="cuda")
    mb.attention_forward(qkv, cud, B, nnz, maxlen, heads, d, sl, Od, lse)
    sp = lambda t: t.reshape(B, Lmax, heads, d)  # noqa: E731
    C, cache = O.attention_forward(sp(qkv_p[..., :H]), sp(qkv_p[..., H:2 * H]), sp(qkv_p[..., 2 * H:]), mask,
                                   slopes_np.astype(np.float64))
    check(f"{case}.O", np64(Od), O.unpad(C.reshape(B, Lmax, H), oidx), max_rel=2e-2)
    q, k, v, P, _ = cache
    s = np.einsum("blhd,bmhd->bhlm", q, k) / np.sqrt(d)
    i = np.arange(Lmax)
    s = s - slopes_np[None, :, None, None] * np.abs(i[:, None] - i[None, :])
    s = np.where(mask[:, None, None, :].astype(bool), s, -np.inf)
    lse_o = np.log(np.exp(s - s.max(-1, keepdims=True)).sum(-1)) + s.max(-1)
    lse_o = np.stack([O.unpad(lse_o[:, h, :], oidx) for h in range(heads)])
    assert np.max(np.abs(np64(lse) - lse_o)) < 2e-2
    dqkv = torch.zeros(nnz, 3 * H, dtype=BF, device="cuda")
    db = torch.zeros(3 * H, dtype=torch.float32, device="cuda")
    mb.attention_backward(qkv, Od, dO, lse, cud, B, nnz, maxlen, heads, d, sl, dqkv, db_qkv=db)
    dq, dk, dv = O.attention_backward(sp(do_p), cache)
    ref = np.concatenate([x.reshape(B, Lmax, H) for x in (dq, dk, dv)], -1)
    ref = O.unpad(ref, oidx)
    got = np64(dqkv)
    for nm, sl_ in (("dq", slice(0, H)), ("dk", slice(H, 2 * H)), ("dv", slice(2 * H, 3 * H))):
        check(f"{case}.{nm}", got[:, sl_], ref[:, sl_])
    # fused bias gradient: column sums of dQKV (db_k is ~0 analytically: rows of dS sum to zero)
    dbref = ref.sum(0)
    check(f"{case}.db_qv", np.concatenate([np64(db)[:H], np64(db)[2 * H:]]),
          np.concatenate([dbref[:H], dbref[2 * H:]]))
    assert np.max(np.abs(np64(db)[H:2 * H])) <= 2e-2 * np.max(np.abs(dbref))


@pytest.mark.parametrize("lo,hi,nseq", [(129, 512, 180), (257, 1024, 60), (1, 128, 400), (1, 40, 500)])
def test_attention_long_many_units(lo, hi, nseq):
    """Several work units per persistent CTA (units > SMs) with ragged lengths: long path with odd
    query-tile counts, and the short path with groups of 4 / pairs / single sequences sharing one
    tile (block-diagonal key windows), zero-length sequences included: exercises the cross-unit
    pipelines (deferred O epilogue, O double-buffering, barrier phases across units).  Oracle per
    sequence (B = 1) to keep host memory small."""
    heads, d = 4, 64
    H = heads * d
    rng = np.random.default_rng(lo + hi)
    lens = rng.integers(lo, hi + 1, size=nseq)
    lens[:3] = [hi, lo, 2 * 128 + 1] if hi > 128 else [hi, lo, 0]
    if hi <= 128:
        lens[10:14] = 0  # a whole empty group
        lens[20] = 0
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    nnz = int(cu[-1])
    qkv_np = synth.bf16_round(rng.standard_normal((nnz, 3 * H)) * 1.5)
    do_np = synth.bf16_round(rng.standard_normal((nnz, H)))
    sl_np = mb.alibi_slopes(heads)
    qkv, dO, cud, sl = _bf(qkv_np), _bf(do_np), to_dev(cu, I32), to_dev(sl_np, torch.float32)
    Od = torch.empty(nnz, H, dtype=BF, device="cuda")
    lse = torch.empty(heads, nnz, dtype=torch.float32, device="cuda")
    mb.attention_forward(qkv, cud, nseq, nnz, int(lens.max()), heads, d, sl, Od, lse)
    dqkv = torch.zeros(nnz, 3 * H, dtype=BF, device="cuda")
    db = torch.zeros(3 * H, dtype=torch.float32, device="cuda")
    mb.attention_backward(qkv, Od, dO, lse, cud, nseq, nnz, int(lens.max()), heads, d, sl, dqkv, db_qkv=db)
    Og, lg, dg = np64(Od), np64(lse), np64(dqkv)
    ref_o, ref_d = np.zeros((nnz, H)), np.zeros((nnz, 3 * H))
    ref_l = np.zeros((heads, nnz))
    for b in range(nseq):
        a, e, L_ = cu[b], cu[b + 1], int(lens[b])
        if L_ == 0:
            continue
        sp = lambda t: t[a:e].reshape(1, L_, heads, d)  # noqa: E731
        C, cache = O.attention_forward(sp(qkv_np[:, :H]), sp(qkv_np[:, H:2 * H]), sp(qkv_np[:, 2 * H:]),
                                       np.ones((1, L_)), sl_np.astype(np.float64))
        ref_o[a:e] = C.reshape(L_, H)
        q, k = cache[0][0], cache[1][0]
        i = np.arange(L_)
        s_ = np.einsum("lhd,mhd->hlm", q, k) / np.sqrt(d) - sl_np[:, None, None] * np.abs(i[:, None] - i[None, :])
        mx = s_.max(-1)
        ref_l[:, a:e] = np.log(np.exp(s_ - mx[..., None]).sum(-1)) + mx
        dq, dk, dv = O.attention_backward(do_np[a:e].reshape(1, L_, heads, d), cache)
        ref_d[a:e] = np.concatenate([x.reshape(L_, H) for x in (dq, dk, dv)], -1)
    check(f"many{hi}.O", Og, ref_o, max_rel=2e-2)
    assert np.max(np.abs(lg - ref_l)) < 2e-2
    for nm, sl_ in (("dq", slice(0, H)), ("dk", slice(H, 2 * H)), ("dv", slice(2 * H, 3 * H))):
        check(f"many{hi}.{nm}", dg[:, sl_], ref_d[:, sl_])


def test_attention_alibi_closed_form():
    """Pin P4b on the kernel: Q = K = 0 -> weights e^{-m|i-j|}/sum (in-kernel bias, masking and the
    per-sequence position restart); l=2, m=ln 3 -> [3/4, 1/4]."""
    heads, d = 2, 32
    H = heads * d
    lens = [2, 5, 7]
    nnz = sum(lens)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    qkv = np.zeros((nnz, 3 * H), np.float32)
    pos = np.concatenate([np.arange(l) for l in lens])
    qkv[:, 2 * H: 2 * H + 1] = pos[:, None]  # v[:, head0, 0] = position
    qkv[:, 2 * H + d: 2 * H + d + 1] = 1.0   # v[:, head1, 0] = 1
    m = np.array([np.log(3.0), 0.5], dtype=np.float32)
    Od = torch.empty(nnz, H, dtype=BF, device="cuda")
    lse = torch.empty(heads, nnz, dtype=torch.float32, device="cuda")
    mb.attention_forward(_bf(qkv), to_dev(cu, I32), 3, nnz, 7, heads, d, to_dev(m, torch.float32), Od, lse)
    out = np64(Od)
    for b, l in enumerate(lens):
        for i in range(l):
            w = np.exp(-float(m[0]) * np.abs(i - np.arange(l)))
            w /= w.sum()
            assert abs(out[cu[b] + i, 0] - np.dot(w, np.arange(l))) < 1e-2 * max(1, l)
            assert abs(out[cu[b] + i, d] - 1.0) < 1e-2
    assert abs(out[0, 0] - 0.25) < 4e-3 and abs(out[1, 0] - 0.75) < 4e-3


# ------------------------------------------------------------------------------------ F3 baselines
@pytest.mark.parametrize("H", [768, 1024])
def test_layernorm_f32_baseline(H):
    """F3 ablation baseline: fp32-activation LayerNorm against the oracle (fp32 storage, so the
    forward is checked at fp32 tolerance)."""
    rng = np.random.default_rng(H + 1)
    n = 517
    x = rng.standard_normal((n, H)).astype(np.float32) * 3 + 1
    g = synth.bf16_round(1 + 0.1 * rng.standard_normal(H))
    b = synth.bf16_round(0.1 * rng.standard_normal(H))
    dy = rng.standard_normal((n, H)).astype(np.float32)
    xd = to_dev(x, torch.float32)
    y = torch.empty(n, H, dtype=torch.float32, device="cuda")
    st = torch.empty(n, 2, dtype=torch.float32, device="cuda")
    mb._lib.layernorm_forward_f32(xd, _bf(g), _bf(b), 1e-12, y, st)
    yo, cache = O.layer_norm(x, g, b, 1e-12)
    check("lnf32.y", np64(y), yo, max_rel=1e-5)
    dx = torch.empty(n, H, dtype=torch.float32, device="cuda")
    dg, dbb, ds = (torch.zeros(H, device="cuda") for _ in range(3))
    mb._lib.layernorm_backward_f32(to_dev(dy, torch.float32), xd, st, _bf(g), dx, dg, dbb, ds)
    dxo, dgo, dbo = O.layer_norm_backward(dy, cache, g)
    check("lnf32.dx", np64(dx), dxo, max_rel=1e-4)
    check("lnf32.dgamma", np64(dg), dgo, max_rel=1e-4)
    check("lnf32.dbeta", np64(dbb), dbo, max_rel=1e-4)
    check("lnf32.dsum", np64(ds), dxo.sum(0), max_rel=1e-3)


def test_geglu_naive_baseline():
    """F3 ablation baseline: the unfused GLU's elementwise kernels against the oracle's GeLU (Eq. 2)."""
    rng = np.random.default_rng(77)
    n, I = 300, 3072
    ua = synth.bf16_round(rng.standard_normal((n, I)) * 2)
    ug = synth.bf16_round(rng.standard_normal((n, I)))
    dz = synth.bf16_round(rng.standard_normal((n, I)))
    z = torch.empty(n, I, dtype=BF, device="cuda")
    mb._lib.geglu_naive_forward(_bf(ua), _bf(ug), z)
    check("geglu_naive.z", np64(z), O.gelu(ua) * ug)
    dua, dug = torch.empty_like(z), torch.empty_like(z)
    mb._lib.geglu_naive_backward(_bf(dz), _bf(ua), _bf(ug), dua, dug)
    check("geglu_naive.dua", np64(dua), dz * ug * O.gelu_grad(ua))
    check("geglu_naive.dug", np64(dug), dz * O.gelu(ua))


# ------------------------------------------------------------------------------------ F1 AdamW
@pytest.mark.parametrize("dev_scale", [False, True])
@pytest.mark.parametrize("n", [1, 7, 1000, 9450243])
def test_adamw_step_vs_oracle(n, dev_scale):
    """mb_adamw_step (decoupled AdamW, R34) against the fp64 oracle over three steps with a changing
    lr / decay factor and a grad_scale: fp32 master, moments within fp32 rounding of the oracle; the
    bf16 weight copy is exactly the RNE of the kernel's own master.  n covers the scalar tail and a
    full Base layer bucket (+3); offset views exercise the unaligned (scalar) path."""
    from paper_2312_17482_b200 import _lib as L
    rng = np.random.default_rng(n)
    w0 = (0.02 * rng.standard_normal(n)).astype(np.float32)
    for off in (0, 1):
        N = n + off
        master = torch.zeros(N, dtype=torch.float32, device="cuda")
        m = torch.zeros_like(master)
        v = torch.zeros_like(master)
        g = torch.zeros_like(master)
        wb = torch.zeros(N, dtype=BF, device="cuda")
        mv, vv, gv, wv = m[off:], v[off:], g[off:], wb[off:]
        pv = master[off:]
        pv.copy_(torch.from_numpy(w0))
        ow, om, ov = w0.astype(np.float64), np.zeros(n), np.zeros(n)
        gmax = 0.0  # moments are sums of terms of size |g'| (g'^2): fp32 rounding is relative to those
        for t in range(1, 4):
            gr = (rng.standard_normal(n) * 10.0 ** rng.integers(-2, 3)).astype(np.float32)
            gmax = max(gmax, float(np.abs(gr).max()) / 3.0)
            gv.copy_(torch.from_numpy(gr))
            lr, wd, gs = 5e-4 * t, 1e-5 * t, 1.0 / 3.0
            if dev_scale:  # the data-parallel form: scale read from device memory (mb_adamw_step_dev)
                L.adamw_step(pv, mv, vv, gv, wv, lr, 0.9, 0.98, 1e-6, wd, 1.0, t,
                             grad_scale_dev=torch.tensor([gs], dtype=torch.float32, device="cuda"))
            else:
                L.adamw_step(pv, mv, vv, gv, wv, lr, 0.9, 0.98, 1e-6, wd, gs, t)
            ow, om, ov = O.adamw_step(ow, om, ov, gr.astype(np.float64), t, lr=lr, wd_step=wd, grad_scale=np.float32(gs))
        torch.cuda.synchronize()
        pg = pv.double().cpu().numpy()
        assert np.allclose(pg, ow, rtol=2e-6, atol=1e-9), float(np.max(np.abs(pg - ow)))
        assert np.allclose(mv.double().cpu().numpy(), om, rtol=2e-6, atol=1e-6 * gmax)
        assert np.allclose(vv.double().cpu().numpy(), ov, rtol=2e-6, atol=1e-6 * gmax * gmax)
        assert torch.equal(wv.cpu(), pv.cpu().to(BF))


# ------------------------------------------------------------------------------------ A3 embedding
@pytest.mark.parametrize("H", [768, 1024])
def test_embedding_fwd_bwd_repeated_ids(H):
    """Embedding gather + LN forward and its backward (dE_tok scatter-add, dE_type, dgamma, dbeta)
    with heavily repeated ids — 60 % of the tokens share one id, like [MASK] in a 30 %-masked
    batch, plus [CLS]/[SEP] at every sequence boundary — so the per-CTA shared-memory accumulation
    of repeated ids carries most of the gradient (H = 1024: its 48 KB configuration)."""
    from paper_2312_17482_b200 import _lib as L
    rng = np.random.default_rng(H)
    B, Lq, V = 64, 128, 30528
    lens = rng.integers(40, Lq + 1, size=B)
    mask = synth.mask_from_lengths(lens, Lq)
    ids = rng.integers(1000, 30522, size=(B, Lq))
    ids[rng.random((B, Lq)) < 0.6] = 103
    ids[:, 0] = 101
    ids[np.arange(B), lens - 1] = 102
    ids = np.where(mask != 0, ids, 0).astype(np.int32)
    emb = synth.bf16_round(0.02 * rng.standard_normal((V, H)))
    typ = synth.bf16_round(0.02 * rng.standard_normal((2, H)))
    g = synth.bf16_round(1 + 0.1 * rng.standard_normal(H))
    b = synth.bf16_round(0.1 * rng.standard_normal(H))
    dX0 = synth.make_grad(mask, H, 3)
    cu, idx, meta = mb.unpad_index(to_dev(mask, I32))
    nnz = int(meta[0].item())
    d = L.dims(H, H // 64, 4 * H, V)
    x0 = torch.empty(nnz, H, dtype=BF, device="cuda")
    st = torch.empty(nnz, 2, dtype=torch.float32, device="cuda")
    ids_d = to_dev(ids, I32)
    L.embed_forward(d, ids_d, idx, nnz, _bf(emb), _bf(typ), _bf(g), _bf(b), x0, st)
    Xo, cache = O.embed_forward(ids, emb, typ, g, b)
    oidx = O.unpad_index(mask)[1]
    check("emb.x0", np64(x0), O.unpad(Xo, oidx))
    dx0 = torch.empty(nnz, H, dtype=BF, device="cuda")
    mb.gather_rows(to_dev(dX0.reshape(B * Lq, H), torch.float32).to(BF), idx, nnz, dx0)
    dE = torch.zeros(V, H, device="cuda")
    dT = torch.zeros(H, device="cuda")
    dg = torch.zeros(H, device="cuda")
    dbb = torch.zeros(H, device="cuda")
    L.embed_backward(d, ids_d, idx, nnz, _bf(emb), _bf(typ), _bf(g), st, dx0, dE, dT, dg, dbb)
    torch.cuda.synchronize()
    dEo, dTo, dgo, dbo = O.embed_backward(dX0, ids, mask, cache, g, V)
    check("emb.dE[MASK]", np64(dE)[103], dEo[103])
    check("emb.dE", np64(dE), dEo)
    check("emb.dtype", np64(dT), dTo[0])
    check("emb.dgamma", np64(dg), dgo)
    check("emb.dbeta", np64(dbb), dbo)


def test_attention_short_huge_batch_fallbacks():
    """More (sequence, head) units than the short kernels' per-CTA unit lists hold (forward: launched
    in chunks of sequences; backward: the long kernel, which takes any length): 80,000 sequences of
    length 1..3."""
    heads, d = 2, 32
    H = heads * d
    rng = np.random.default_rng(80000)
    B, Lmax = 80000, 3
    lens = rng.integers(1, Lmax + 1, size=B)
    mask = synth.mask_from_lengths(lens, Lmax)
    qkv_p = synth.bf16_round(rng.standard_normal((B, Lmax, 3 * H)))
    do_p = synth.bf16_round(rng.standard_normal((B, Lmax, H))) * mask[..., None]
    cu, oidx, maxlen, _ = O.unpad_index(mask)
    nnz = len(oidx)
    sl_np = mb.alibi_slopes(heads)
    qkv, dO, cud, sl = _bf(O.unpad(qkv_p, oidx)), _bf(O.unpad(do_p, oidx)), to_dev(cu, I32), to_dev(sl_np, torch.float32)
    Od = torch.empty(nnz, H, dtype=BF, device="cuda")
    lse = torch.empty(heads, nnz, dtype=torch.float32, device="cuda")
    mb.attention_forward(qkv, cud, B, nnz, maxlen, heads, d, sl, Od, lse)
    dqkv = torch.zeros(nnz, 3 * H, dtype=BF, device="cuda")
    mb.attention_backward(qkv, Od, dO, lse, cud, B, nnz, maxlen, heads, d, sl, dqkv)
    sp = lambda t: t.reshape(B, Lmax, heads, d)  # noqa: E731
    C, cache = O.attention_forward(sp(qkv_p[..., :H]), sp(qkv_p[..., H:2 * H]), sp(qkv_p[..., 2 * H:]), mask,
                                   sl_np.astype(np.float64))
    check("huge.O", np64(Od), O.unpad(C.reshape(B, Lmax, H), oidx), max_rel=2e-2)
    dq, dk, dv = O.attention_backward(sp(do_p), cache)
    ref = O.unpad(np.concatenate([x.reshape(B, Lmax, H) for x in (dq, dk, dv)], -1), oidx)
    got = np64(dqkv)
    for nm, s_ in (("dq", slice(0, H)), ("dk", slice(H, 2 * H)), ("dv", slice(2 * H, 3 * H))):
        check(f"huge.{nm}", got[:, s_], ref[:, s_])


def test_attention_short_forward_chunked_launches():
    """The short forward launches batches beyond num_sms x 96 units in chunks of sequences (offsets
    into cu_seqlens): 1,200 sequences x 12 heads, lengths 90..128, so the second launch holds a ragged
    remainder and full-quarter tiles take the TMA-staged output path in both launches."""
    heads, d = 12, 32
    H = heads * d
    rng = np.random.default_rng(1200)
    B, Lmax = 1200, 128
    lens = rng.integers(90, Lmax + 1, size=B)
    lens[-1] = Lmax
    mask = synth.mask_from_lengths(lens, Lmax)
    qkv_p = synth.bf16_round(rng.standard_normal((B, Lmax, 3 * H)))
    cu, oidx, maxlen, _ = O.unpad_index(mask)
    nnz = len(oidx)
    sl_np = mb.alibi_slopes(heads)
    qkv, cud, sl = _bf(O.unpad(qkv_p, oidx)), to_dev(cu, I32), to_dev(sl_np, torch.float32)
    Od = torch.empty(nnz, H, dtype=BF, device="cuda")
    lse = torch.empty(heads, nnz, dtype=torch.float32, device="cuda")
    mb.attention_forward(qkv, cud, B, nnz, maxlen, heads, d, sl, Od, lse)
    sp = lambda t: t.reshape(B, Lmax, heads, d)  # noqa: E731
    C, _ = O.attention_forward(sp(qkv_p[..., :H]), sp(qkv_p[..., H:2 * H]), sp(qkv_p[..., 2 * H:]), mask,
                               sl_np.astype(np.float64))
    check("chunked.O", np64(Od), O.unpad(C.reshape(B, Lmax, H), oidx), max_rel=2e-2)
