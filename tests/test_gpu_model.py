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


def _layer_parity(dims, lens, Lmax, regime, seed):
    H, n = dims.hidden, dims.heads
    p = synth.make_layer_params(dims, seed, regime)
    mask = synth.mask_from_lengths(np.array(lens), Lmax)
    X = synth.make_hidden(mask, H, seed + 1)
    dY = synth.make_grad(mask, H, seed + 2)
    Y, c = O.encoder_layer_forward(X, mask, O.alibi_slopes(n), p, dims.ln_eps)
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
    mb.encoder_forward(cd, pd, pk, slopes, x, y, saved)
    dy = torch.empty_like(x)
    mb.gather_rows(to_dev(dY.reshape(B * Lmax, H), torch.float32).to(BF), idx, nnz, dy)
    dx = torch.empty_like(x)
    ws = torch.empty(L.layer_workspace_bytes(cd, nnz, maxlen), dtype=torch.uint8, device="cuda")
    mb.encoder_backward(cd, pd, pk, slopes, x, saved, dy, dx, gd, ws)
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


def test_layer_large_dims():
    _layer_parity(synth.LARGE, [128, 128, 40], 128, "stress", 6)


def _model_parity(dims, batch, params, tol_loss=1e-2):
    model = mb.MosaicBert(mb.ModelDims(dims.hidden, dims.heads, dims.intermediate, dims.vocab,
                                       len(params["layers"]), dims.ln_eps), params)
    n_lab = int(((batch["labels"] != -100) & (batch["attention_mask"] != 0)).sum())
    model.zero_grad()
    ids, mask, labels = (to_dev(batch[k], I32) for k in ("input_ids", "attention_mask", "labels"))
    model.micro_step(ids, mask, labels, inv_norm=1.0 / n_lab)
    torch.cuda.synchronize()
    loss = float(model.loss_sum.item())
    oloss, og = O.model_forward_backward(batch, params, O.alibi_slopes(dims.heads), dims.ln_eps)
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


def test_loss_zero_decoder_is_lnV():
    """Pin P12 on the GPU path: E_tok = 0 and b_dec = 0 give loss = ln V exactly (up to fp32)."""
    params = synth.make_model_params(synth.TINY, 3, "stress")
    params["emb"] = np.zeros_like(params["emb"])
    params["b_dec"] = np.zeros_like(params["b_dec"])
    batch = synth.make_batch("C1", 8)
    loss, _ = _model_parity(synth.TINY, batch, params, tol_loss=1e-5)
    assert abs(loss - np.log(128)) < 1e-5
