"""P18: the oracle's WHOLE-MODEL step at full depth (12 and 24 layers, the Base / Large layer counts
of BASELINE configs 2-5, at tiny widths) against an independent torch-CPU-fp64 autograd
re-implementation built from library primitives (F.embedding, F.layer_norm,
F.scaled_dot_product_attention with the ALiBi float mask, F.gelu, F.cross_entropy): loss and every
parameter gradient.  This pins the composition — layer chaining, the tied decoder / embedding
gradient sum (R15), the R18 normaliser — at the depths the GPU step runs, which the per-layer pins
(P13/P14) and the 1-layer model finite differences do not reach."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O
import synth
from test_oracle_grad import _torch_layer

pytestmark = pytest.mark.filterwarnings("ignore")


def _torch_model(batch, params, slopes, eps):
    t = lambda a: torch.tensor(np.asarray(a, dtype=np.float64), requires_grad=True)  # noqa: E731
    tp = {k: t(v) for k, v in params.items() if k != "layers"}
    tl = [{k: t(v) for k, v in lp.items()} for lp in params["layers"]]
    ids = torch.tensor(batch["input_ids"].astype(np.int64))
    mask = batch["attention_mask"]
    labels = batch["labels"].astype(np.int64)
    H = tp["emb"].shape[1]
    X = F.layer_norm(F.embedding(ids, tp["emb"]) + F.embedding(torch.zeros_like(ids), tp["type_emb"]), (H,),
                     tp["lne_g"], tp["lne_b"], eps)
    for lp in tl:
        X = _torch_layer(X, mask, slopes, lp, eps)
    sel = torch.from_numpy((labels != -100) & (mask != 0))
    h = F.gelu(F.linear(X[sel], tp["w_t"], tp["b_t"]))
    u = F.layer_norm(h, (H,), tp["lnh_g"], tp["lnh_b"], eps)
    z = F.linear(u, tp["emb"], tp["b_dec"])
    y = torch.from_numpy(labels)[sel]
    loss = F.cross_entropy(z, y, reduction="sum") / int(sel.sum())
    loss.backward()
    return loss.item(), tp, tl


@pytest.mark.parametrize("n_layers,regime", [(12, "stress"), (12, "bert"), (24, "stress")])
def test_p18_full_depth_model_matches_torch(n_layers, regime):
    dims = synth.TINY
    params = synth.make_model_params(dims, 40 + n_layers, regime, n_layers=n_layers)
    params = {k: (v.astype(np.float64) if k != "layers" else
                  [{kk: vv.astype(np.float64) for kk, vv in l.items()} for l in v]) for k, v in params.items()}
    batch = synth.make_batch("C1", 70 + n_layers)
    slopes = O.alibi_slopes(dims.heads)
    eps = 1e-12
    loss, grads = O.model_forward_backward(batch, params, slopes, eps)
    tloss, tp, tl = _torch_model(batch, params, slopes, eps)
    assert abs(loss - tloss) <= 1e-10 * max(1.0, abs(tloss)), (loss, tloss)

    def close(a, ref, name):
        scale = max(1e-30, float(np.abs(ref).max()))
        err = float(np.abs(a - ref).max()) / scale
        assert err <= 1e-9, (name, err)

    for k, v in tp.items():
        close(grads[k], v.grad.numpy(), k)
    assert len(grads["layers"]) == n_layers
    for li, lp in enumerate(tl):
        for k, v in lp.items():
            close(grads["layers"][li][k], v.grad.numpy(), f"L{li}.{k}")
