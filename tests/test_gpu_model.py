"""GPU parity at the layer and model level: the packed CUDA path (mb_encoder_forward/backward,
mb_embed_*, mb_mlm_loss through the MosaicBert driver) against the fp64 oracle on the PADDED batch,
compared on the real rows."""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from parity import check, np64, to_dev

pytestmark = pytest.mark.gpu
mb = pytest.importorskip("paper_2312_17482_b200")
from paper_2312_17482_b200 import _lib as L  # noqa: E402

BF = torch.bfloat16
I32 = torch.int32


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mb.lib()


def _layer_parity(dims, lens, Lmax, regime, seed, dropout=None):
    """dropout: None or dict(p, seed, stream) (F2, R32) — the same mask is regenerated on both sides."""
    H, n = dims.hidden, dims.heads
    p = synth.make_layer_params(dims, seed, regime)
    mask = synth.mask_from_lengths(np.array(lens), Lmax)
    X = synth.make_hidden(mask, H, seed + 1)
    dY = synth.make_grad(mask, H, seed + 2)
    Y, c = O.encoder_layer_forward(X, mask, O.alibi_slopes(n), p, dims.ln_eps, dropout)
    drop = L.Dropout(dropout["p"], dropout["seed"], dropout["stream"]) if dropout else None
    dX, g = O.encoder_layer_backward(dY, c)
    B = len(lens)
    cu, idx, meta = mb.unpad_index(to_dev(mask, I32))
    nnz, maxlen = (int(v) for v in meta[:2].tolist())
    cd = L.dims(H, n, dims.intermediate, dims.vocab, dims.ln_eps)
    pk = L.Packed(cu.data_ptr(), B, nnz, maxlen)
    pd = {k: to_dev(v, torch.float32).to(BF) for k, v in p.items()}
    gd = {k: torch.zeros(v.shape, dtype=torch.float32, device="cuda") for k, v in p.items()}
    slopes = to_dev(mb.alibi_slopes(n), torch.float32)
    x = torch.empty(nnz, H, dtype=BF, device="cuda")
    mb.gather_rows(to_dev(X.reshape(B * Lmax, H), torch.float32).to(BF), idx, nnz, x)
    y = torch.empty_like(x)
    saved = torch.empty(L.layer_saved_bytes(cd, nnz), dtype=torch.uint8, device="cuda")
    mb.encoder_forward(cd, pd, pk, slopes, x, y, saved, drop)
    dy = torch.empty_like(x)
    mb.gather_rows(to_dev(dY.reshape(B * Lmax, H), torch.float32).to(BF), idx, nnz, dy)
    dx = torch.empty_like(x)
    ws = torch.empty(L.layer_workspace_bytes(cd, nnz, maxlen), dtype=torch.uint8, device="cuda")
    mb.encoder_backward(cd, pd, pk, slopes, x, saved, dy, dx, gd, ws, drop)
    torch.cuda.synchronize()
    oidx = O.unpad_index(mask)[1]
    check("layer.Y", np64(y), O.unpad(Y, oidx))
    check("layer.dX", np64(dx), O.unpad(dX, oidx))
    for k in p:
        check(f"layer.d{k}", np64(gd[k]), g[k])


@pytest.mark.parametrize("regime", ["stress", "bert"])
@pytest.mark.parametrize("seed", [0, 1])
def test_layer_tiny(regime, seed):
    _layer_parity(synth.TINY, [16, 9, 3, 1], 16, regime, seed)


@pytest.mark.parametrize("regime", ["stress", "bert"])
def test_layer_base_dims_ragged(regime):
    lens = synth.make_lengths("lognormal", 12, 128, synth.rng_for(5))
    lens[0] = 128
    _layer_parity(synth.BASE, list(lens), 128, regime, 3)


def test_layer_base_seq512():
    _layer_parity(synth.BASE, [512, 300, 129], 512, "stress", 4)


def test_layer_base_seq1024():
    """F4: a Base layer at l = 1024 (ragged second sequence)."""
    _layer_parity(synth.BASE, [1024, 517], 1024, "bert", 12)


def test_layer_large_dims():
    _layer_parity(synth.LARGE, [128, 128, 40], 128, "stress", 6)


# ----------------------------------------------------------------------------- F2 dropout (R32)
@pytest.mark.parametrize("site", [0, 1])
@pytest.mark.parametrize("p", [0.1, 0.5])
def test_dropout_mask_bitexact(site, p):
    """The device Philox mask (the function the fused epilogues call) equals the oracle's, bit for
    bit, including a 64-bit seed whose high word matters and a ragged row count."""
    from oracle.philox import dropout_keep
    rows, cols, seed, stream = 1003, 768, (1 << 40) + 12345, 7
    out = torch.empty(rows, cols, dtype=torch.uint8, device="cuda")
    L.dropout_mask(L.Dropout(p, seed, stream), site, rows, cols, out)
    torch.cuda.synchronize()
    ref = dropout_keep(rows, cols, p, seed, stream, site)
    assert np.array_equal(out.cpu().numpy().astype(bool), ref)


@pytest.mark.parametrize("regime", ["stress", "bert"])
def test_layer_tiny_dropout(regime):
    _layer_parity(synth.TINY, [16, 9, 3, 1], 16, regime, 2, dict(p=0.1, seed=77, stream=1))


def test_layer_base_dropout_ragged():
    lens = synth.make_lengths("lognormal", 12, 128, synth.rng_for(7))
    lens[0] = 128
    _layer_parity(synth.BASE, list(lens), 128, "bert", 8, dict(p=0.1, seed=(3 << 33) + 5, stream=11))


def test_layer_base_dropout_high_p():
    """p = 0.5 makes any mask disagreement between the epilogue / LN-backward and the oracle large."""
    _layer_parity(synth.BASE, [128, 77, 128], 128, "stress", 9, dict(p=0.5, seed=4242, stream=0))


def _model_parity(dims, batch, params, tol_loss=1e-2, dropout=None):
    model = mb.MosaicBert(mb.ModelDims(dims.hidden, dims.heads, dims.intermediate, dims.vocab,
                                       len(params["layers"]), dims.ln_eps), params,
                          dropout=dropout["p"] if dropout else 0.0)
    n_lab = int(((batch["labels"] != -100) & (batch["attention_mask"] != 0)).sum())
    model.zero_grad()
    ids, mask, labels = (to_dev(batch[k], I32) for k in ("input_ids", "attention_mask", "labels"))
    model.micro_step(ids, mask, labels, inv_norm=1.0 / n_lab, drop_seed=dropout["seed"] if dropout else None)
    torch.cuda.synchronize()
    loss = float(model.loss_sum.item())
    oloss, og = O.model_forward_backward(batch, params, O.alibi_slopes(dims.heads), dims.ln_eps, dropout=dropout)
    assert abs(loss - oloss) <= tol_loss, (loss, oloss)
    gg = model.grads_numpy()
    for k in ("emb", "type_emb", "lne_g", "lne_b", "w_t", "b_t", "lnh_g", "lnh_b", "b_dec"):
        check(f"model.d{k}", gg[k], og[k])
    for li, (a, b) in enumerate(zip(gg["layers"], og["layers"])):
        for k in b:
            check(f"model.L{li}.d{k}", a[k], b[k])
    return loss, oloss


@pytest.mark.parametrize("regime", ["stress", "bert"])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_model_step_c1(regime, seed):
    params = synth.make_model_params(synth.TINY, seed, regime)
    batch = synth.make_batch("C1", 100 + seed)
    _model_parity(synth.TINY, batch, params)


def test_model_step_base_two_layers():
    """Base dims (V = 30528 head, 12 heads) with 2 layers and a C5-like ragged batch."""
    params = synth.make_model_params(synth.BASE, 9, "bert", n_layers=2)
    batch = synth.make_batch("C5", 5001, B=6)
    _model_parity(synth.BASE, batch, params)


@pytest.mark.parametrize("seed", [0, 1])
def test_model_step_c1_dropout(seed):
    params = synth.make_model_params(synth.TINY, 20 + seed, "bert")
    batch = synth.make_batch("C1", 300 + seed)
    _model_parity(synth.TINY, batch, params, dropout=dict(p=0.1, seed=555 + seed))


def test_model_step_vocab_30522():
    """F3: the unpadded BERT vocabulary (30522, not a multiple of 8 or 64 — P:174) through the
    decoder/CE GEMMs (ragged last column vector, padded dz rows) and the bucket layout."""
    import dataclasses
    dims = dataclasses.replace(synth.BASE, vocab=30522)
    params = synth.make_model_params(dims, 10, "bert", n_layers=2)
    batch = synth.make_batch("C5", 5003, B=6)
    assert batch["input_ids"].max() < 30522
    _model_parity(dims, batch, params)


def test_model_step_degenerate_batches():
    """Edge cases of one micro-step: no labelled token (loss 0, every gradient exactly 0 — the
    head writes a zero upstream gradient) and an all-padding batch (nothing to do)."""
    params = synth.make_model_params(synth.TINY, 4, "stress")
    dims = synth.TINY
    model = mb.MosaicBert(mb.ModelDims(dims.hidden, dims.heads, dims.intermediate, dims.vocab, 1, dims.ln_eps), params)
    batch = synth.make_batch("C1", 77)
    labels = np.full_like(batch["labels"], -100)
    model.zero_grad()
    nnz, n_m = model.micro_step(*(to_dev(x, I32) for x in (batch["input_ids"], batch["attention_mask"], labels)))
    torch.cuda.synchronize()
    assert nnz == int(batch["attention_mask"].sum()) and n_m == 0
    assert float(model.loss_sum.item()) == 0.0
    assert all(float(b.g.abs().max().item()) == 0.0 for b in model.buckets)
    empty = np.zeros_like(batch["attention_mask"])
    model.zero_grad()
    nnz, n_m = model.micro_step(*(to_dev(x, I32) for x in (batch["input_ids"], empty, batch["labels"])))
    torch.cuda.synchronize()
    assert (nnz, n_m) == (0, 0)
    assert all(float(b.g.abs().max().item()) == 0.0 for b in model.buckets)


def test_loss_zero_decoder_is_lnV():
    """Pin P12 on the GPU path: E_tok = 0 and b_dec = 0 give loss = ln V exactly (up to fp32)."""
    params = synth.make_model_params(synth.TINY, 3, "stress")
    params["emb"] = np.zeros_like(params["emb"])
    params["b_dec"] = np.zeros_like(params["b_dec"])
    batch = synth.make_batch("C1", 8)
    loss, _ = _model_parity(synth.TINY, batch, params, tol_loss=1e-5)
    assert abs(loss - np.log(128)) < 1e-5


def test_host_meta_path_matches_and_is_checked():
    """train_step(host_meta=...) skips the device->host read of the unpad results: same loss and
    gradients as the synchronising path; a wrong host value is caught by the deferred check."""
    params = synth.make_model_params(synth.TINY, 6, "stress")
    dims = synth.TINY
    model = mb.MosaicBert(mb.ModelDims(dims.hidden, dims.heads, dims.intermediate, dims.vocab, 1, dims.ln_eps), params)
    batch = synth.make_batch("C1", 41)
    dev = tuple(to_dev(batch[k], I32) for k in ("input_ids", "attention_mask", "labels"))
    meta = mb.MosaicBert.batch_meta(batch["attention_mask"], batch["labels"])
    assert meta[0] == int(batch["attention_mask"].sum())
    l0 = float(model.train_step([dev], optimizer=False).item())
    g0 = model.grads_numpy()
    l1 = float(model.train_step([dev], optimizer=False, host_meta=[meta]).item())
    model.check_meta()
    g1 = model.grads_numpy()
    assert abs(l0 - l1) <= 1e-6 * abs(l0)
    for k in ("emb", "w_t", "b_dec"):
        check(f"host_meta.d{k}", g1[k], g0[k], max_rel=1e-5, min_cos=0.999999)
    # (one masked row fewer: a wrong value that still only touches valid rows)
    model.train_step([dev], optimizer=False, host_meta=[(meta[0], meta[1], meta[2] - 1)])
    with pytest.raises(RuntimeError, match="host batch metadata"):
        model.check_meta()


def test_training_memorises_one_batch():
    """End-to-end sanity of the whole train step (forward, backward, allreduce-free DP path,
    decoupled AdamW with the bf16 weight copy): repeated steps on one tiny batch drive its MLM
    loss far below the initial ln(V)-level value."""
    params = synth.make_model_params(synth.TINY, 11, "bert")
    dims = synth.TINY
    model = mb.MosaicBert(mb.ModelDims(dims.hidden, dims.heads, dims.intermediate, dims.vocab, 1, dims.ln_eps),
                          params, lr_peak=3e-3)
    batch = synth.make_batch("C1", 2024, B=8)
    dev = tuple(to_dev(batch[k], I32) for k in ("input_ids", "attention_mask", "labels"))
    meta = mb.MosaicBert.batch_meta(batch["attention_mask"], batch["labels"])
    losses = [float(model.train_step([dev], host_meta=[meta]).item()) for _ in range(80)]
    model.check_meta()
    assert all(np.isfinite(losses))
    assert losses[0] > 0.8 * np.log(dims.vocab), losses[0]
    assert losses[-1] < 0.25 * losses[0], (losses[0], losses[-1])


def test_model_step_with_empty_rows():
    """Zero-length rows inside a batch (R5: allowed, they have no queries): the packed stream skips
    them in every kernel (attention units, index scans, head) and the step matches the oracle."""
    params = synth.make_model_params(synth.TINY, 12, "stress")
    batch = synth.make_batch("C1", 512, B=6, lengths=np.array([16, 0, 5, 0, 1, 9]))
    assert batch["attention_mask"][1].sum() == 0 and batch["attention_mask"][3].sum() == 0
    _model_parity(synth.TINY, batch, params)


def test_model_step_large_dims_one_layer():
    """MosaicBERT-Large widths (H = 1024, 16 heads, GLU 4096, V = 30528) through embedding (the
    H = 1024 embedding backward with its 48 KB shared-memory accumulators), one layer and the head."""
    params = synth.make_model_params(synth.LARGE, 13, "bert", n_layers=1)
    batch = synth.make_batch("C3", 5013, B=4)
    _model_parity(synth.LARGE, batch, params)


def test_host_meta_growing_batch():
    """with host_meta, a later micro-batch larger than any earlier one regrows the
    buffers; the deferred check of the previous micro-step must still read ITS metadata."""
    params = synth.make_model_params(synth.TINY, 6, "stress")
    dims = synth.TINY
    model = mb.MosaicBert(mb.ModelDims(dims.hidden, dims.heads, dims.intermediate, dims.vocab, 1, dims.ln_eps), params)
    small = synth.make_batch("C1", 41, B=4, L=16)
    big = synth.make_batch("C1", 42, B=8, L=24)
    mbs, metas = [], []
    for b in (small, big, small):
        mbs.append(tuple(to_dev(b[k], I32) for k in ("input_ids", "attention_mask", "labels")))
        metas.append(mb.MosaicBert.batch_meta(b["attention_mask"], b["labels"]))
    loss = float(model.train_step(mbs, optimizer=False, host_meta=metas).item())
    model.check_meta()
    ref = float(mb.MosaicBert(mb.ModelDims(dims.hidden, dims.heads, dims.intermediate, dims.vocab, 1, dims.ln_eps),
                              params).train_step(mbs, optimizer=False).item())
    assert abs(loss - ref) <= 1e-6 * abs(ref)


def test_token_id_range_reported_and_clamped():
    """an id outside [0, V) at a REAL position is reported by mb_unpad_index
    (MB_ERR_TOKEN_RANGE in meta[2]); at a pad position it is ignored; the embedding kernels clamp, so
    nothing outside E_tok / dE_tok is touched, and the model step rejects the batch."""
    dims = synth.TINY
    batch = synth.make_batch("C1", 77)
    mask = batch["attention_mask"]
    ids = batch["input_ids"].copy()
    b = int(np.argmin(mask.sum(1)))
    ids[b, -1] = 10_000 if mask[b, -1] == 0 else ids[b, -1]  # pad position: ignored
    _, _, meta = mb.unpad_index(to_dev(mask, I32), ids=to_dev(ids, I32), vocab=dims.vocab)
    assert int(meta[2]) == 0
    for bad in (-1, dims.vocab):
        ids2 = ids.copy()
        ids2[0, 0] = bad  # row 0 is a full row: position 0 is real
        _, _, meta = mb.unpad_index(to_dev(mask, I32), ids=to_dev(ids2, I32), vocab=dims.vocab)
        assert L.STATUS[int(meta[2])] == "MB_ERR_TOKEN_RANGE"
        # the mask-layout error takes precedence
        m2 = mask.copy()
        m2[0, 1] = 0
        _, _, meta = mb.unpad_index(to_dev(m2, I32), ids=to_dev(ids2, I32), vocab=dims.vocab)
        assert L.STATUS[int(meta[2])] == "MB_ERR_MASK_LAYOUT"
    params = synth.make_model_params(dims, 1, "stress")
    model = mb.MosaicBert(mb.ModelDims(dims.hidden, dims.heads, dims.intermediate, dims.vocab, 1, dims.ln_eps), params)
    ids2 = ids.copy()
    ids2[0, 0] = dims.vocab + 5
    guard = model.emb_bucket.g.clone()
    with pytest.raises(RuntimeError, match="TOKEN_RANGE"):
        model.train_step([(to_dev(ids2, I32), to_dev(mask, I32), to_dev(batch["labels"], I32))], optimizer=False)
    assert torch.equal(model.emb_bucket.g, guard)  # rejected before any kernel wrote a gradient


def test_unpad_select_workspace_and_concurrent_streams():
    """The index scans use only the caller's workspace: the single-CTA (no workspace) and multi-CTA
    kernels agree bit for bit, and two streams running mb_unpad_index / mb_mlm_select concurrently on
    different batches (their own workspaces) both stay bit-exact vs the oracle."""
    cases = [synth.make_batch("C5", 3100 + i, B=512) for i in range(2)]
    s = [torch.cuda.Stream() for _ in cases]
    dev = [(to_dev(c["attention_mask"], I32), to_dev(c["labels"], I32).reshape(-1)) for c in cases]
    outs = [None, None]
    torch.cuda.synchronize()
    for i, (m, lab) in enumerate(dev):
        with torch.cuda.stream(s[i]):
            count = torch.zeros(1, dtype=torch.float32, device="cuda")
            cu, idx, meta = mb.unpad_index(m)
            rows, labs = mb.mlm_select(lab, idx, synth.BASE.vocab, meta, count=count)
            outs[i] = (cu, idx, meta, rows, labs, count)
    torch.cuda.synchronize()
    for c, (cu, idx, meta, rows, labs, count) in zip(cases, outs):
        ocu, oidx, omax, ost = O.unpad_index(c["attention_mask"])
        nnz, mx, st, n_m = (int(v) for v in meta.tolist())
        assert (nnz, mx, st) == (len(oidx), omax, ost)
        assert np.array_equal(cu.cpu().numpy(), ocu) and np.array_equal(idx.cpu().numpy()[:nnz], oidx)
        lab = c["labels"].reshape(-1)[oidx]
        sel = np.flatnonzero(lab != -100)
        assert n_m == len(sel) and float(count.item()) == n_m
        assert np.array_equal(rows.cpu().numpy()[:n_m], sel) and np.array_equal(labs.cpu().numpy()[:n_m], lab[sel])
        # the workspace-free single-CTA kernels give the same bits
        m = to_dev(c["attention_mask"], I32)
        cu1, idx1, meta1 = mb.unpad_index(m, ws=False)
        rows1, labs1 = mb.mlm_select(to_dev(c["labels"], I32).reshape(-1), idx1, synth.BASE.vocab, meta1, ws=False)
        assert torch.equal(cu1, cu) and torch.equal(idx1[:nnz], idx[:nnz]) and torch.equal(meta1, meta)
        assert torch.equal(rows1[:n_m], rows[:n_m]) and torch.equal(labs1[:n_m], labs[:n_m])


def test_loss_normalize_device_count():
    """R18 on the device: inv = 1 / max(N, 1), loss = loss_sum * inv, N from a device scalar or the host."""
    ls = torch.tensor([12.5], device="cuda")
    inv, out = torch.zeros(1, device="cuda"), torch.zeros(1, device="cuda")
    mb.loss_normalize(ls, count=torch.tensor([5.0], device="cuda"), inv_out=inv, loss_out=out)
    assert float(inv) == np.float32(1 / 5.0) and abs(float(out) - 2.5) < 1e-6
    mb.loss_normalize(ls, count_host=0.0, inv_out=inv, loss_out=out)
    assert float(inv) == 1.0 and float(out) == 12.5


def test_evaluate_matches_training_forward():
    """MosaicBert.evaluate (forward only, mb_mlm_loss with dy_top = grads = NULL) runs exactly the
    training step's forward kernels: the summed loss is bitwise the micro-step's, and the training
    state (gradients, R18 count, loss accumulator) is untouched by it."""
    params = synth.make_model_params(synth.TINY, 4, "bert")
    batch = synth.make_batch("C1", 77)
    d = synth.TINY
    model = mb.MosaicBert(mb.ModelDims(d.hidden, d.heads, d.intermediate, d.vocab, 1, d.ln_eps), params)
    ids, mask, labels = (to_dev(batch[k], I32) for k in ("input_ids", "attention_mask", "labels"))
    n_lab = int(((batch["labels"] != -100) & (batch["attention_mask"] != 0)).sum())
    model.zero_grad()
    model.micro_step(ids, mask, labels, inv_norm=1.0)
    torch.cuda.synchronize()
    ref_loss = float(model.loss_sum.item())
    ref_g = [b.g.clone() for b in model.buckets]
    ref_count = float(model.count_dev.item())
    s_eval, n_eval = model.evaluate(ids, mask, labels)
    assert n_eval == n_lab
    assert s_eval == ref_loss, (s_eval, ref_loss)
    assert float(model.loss_sum.item()) == ref_loss and float(model.count_dev.item()) == ref_count
    assert all(torch.equal(a, b.g) for a, b in zip(ref_g, model.buckets))


@pytest.mark.parametrize("Lq,lens", [(512, [512, 300, 129, 1]), (1024, [1024, 515, 64]), (2048, [2048, 700])])
def test_evaluate_long_sequences_vs_oracle(Lq, lens):
    """SURVEY F4 "train short, test long" (ALiBi lets a model trained at 128 run at longer l):
    the same weights evaluated forward-only at l up to 2048 (the long attention kernels) give the
    oracle's mean MLM loss within the north_star loss bar."""
    d = synth.TINY
    params = synth.make_model_params(d, 6, "bert")
    batch = synth.make_batch("C1", 900 + Lq, B=len(lens), L=Lq, lengths=np.array(lens))
    model = mb.MosaicBert(mb.ModelDims(d.hidden, d.heads, d.intermediate, d.vocab, 1, d.ln_eps), params)
    ids, mask, labels = (to_dev(batch[k], I32) for k in ("input_ids", "attention_mask", "labels"))
    s_eval, n = model.evaluate(ids, mask, labels)
    oloss, _ = O.model_forward_backward(batch, params, O.alibi_slopes(d.heads), d.ln_eps)
    assert n > 0 and abs(s_eval / n - oloss) <= 1e-2, (s_eval / n, oloss)
