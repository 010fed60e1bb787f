"""Data-parallel path on CPU with world_size 2 (gloo): the product's bucketed gradient allreduce and
global masked-count normalisation (model.MosaicBert, R18) must turn per-shard gradients into the
gradient of the whole global batch (SURVEY §8e invariant).  Per-shard gradients come from the oracle
(test infrastructure); the reduction and scaling are the product's code."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard(batch, rank, world):
    B = batch["input_ids"].shape[0]
    per = B // world
    return {k: v[rank * per:(rank + 1) * per] for k, v in batch.items()}


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2312_17482_b200.model import ModelDims, MosaicBert
    d = synth.TINY
    params = synth.make_model_params(d, 4, "stress")
    batch = synth.make_batch("C1", 77, B=8)
    shard = _shard(batch, rank, world)
    model = MosaicBert(ModelDims(d.hidden, d.heads, d.intermediate, d.vocab, d.layers), params, device="cpu")
    # per-shard Sigma-loss gradients (inv_norm = 1), as the GPU micro-step produces them
    _, g = O.model_forward_backward(shard, params, O.alibi_slopes(d.heads), inv_norm=1.0)
    for b, lg in zip(model.layer_buckets, g["layers"]):
        for k, v in lg.items():
            b.gv[k].copy_(torch.from_numpy(v))
    for b in (model.head_bucket, model.emb_bucket):
        for k in b.gv:
            b.gv[k].copy_(torch.from_numpy(g[k]))
    n_local = int(((shard["labels"] != -100) & (shard["attention_mask"] != 0)).sum())
    n_global = model.global_masked(n_local)
    model.allreduce_grads()
    model.wait_grads()
    scale = 1.0 / n_global
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), n_global=n_global,
             **{f"L0_{k}": v.numpy() * scale for k, v in model.layer_buckets[0].gv.items()},
             **{k: v.numpy() * scale for b in (model.head_bucket, model.emb_bucket) for k, v in b.gv.items()})
    dist.destroy_process_group()


def test_dp_world2_gradient_equivalence(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    d = synth.TINY
    params = synth.make_model_params(d, 4, "stress")
    batch = synth.make_batch("C1", 77, B=8)
    n_all = int(((batch["labels"] != -100) & (batch["attention_mask"] != 0)).sum())
    _, full = O.model_forward_backward(batch, params, O.alibi_slopes(d.heads))  # mean over the global batch
    r0, r1 = (np.load(tmp_path / f"r{r}.npz") for r in range(world))
    assert int(r0["n_global"]) == n_all == int(r1["n_global"])
    for k, v in full["layers"][0].items():
        assert np.allclose(r0[f"L0_{k}"], v, rtol=1e-5, atol=1e-6 * np.abs(v).max()), k
        assert np.array_equal(r0[f"L0_{k}"], r1[f"L0_{k}"]), k  # every rank holds the same reduced gradient
    for k in ("emb", "type_emb", "lne_g", "w_t", "b_t", "lnh_g", "b_dec"):
        assert np.allclose(r0[k], full[k], rtol=1e-5, atol=1e-6 * np.abs(full[k]).max()), k


def test_optimizer_waits_each_bucket_in_issue_order(monkeypatch):
    """The DP optimizer step updates the buckets in the order their allreduces were issued (head,
    layers last to first, embedding), each only after waiting for its own reduction, so the last
    bucket's transfer overlaps the other updates; buckets without a pending reduction follow."""
    from paper_2312_17482_b200 import _lib as L
    from paper_2312_17482_b200.model import ModelDims, MosaicBert
    d = synth.TINY
    model = MosaicBert(ModelDims(d.hidden, d.heads, d.intermediate, d.vocab, 2), synth.make_model_params(d, 1, n_layers=2),
                       device="cpu")
    log = []

    class Work:
        def __init__(self, name):
            self.name = name

        def wait(self):
            log.append(("wait", self.name))

    names = {id(model.head_bucket): "head", id(model.emb_bucket): "emb",
             id(model.layer_buckets[0]): "L0", id(model.layer_buckets[1]): "L1"}
    model._handles = [(b, Work(names[id(b)])) for b in (model.head_bucket, model.layer_buckets[1], model.emb_bucket)]
    monkeypatch.setattr(L, "adamw_step", lambda master, *a, **k: log.append(("adam", next(
        n for b in model.buckets for n in [names[id(b)]] if b.master is master))))
    model.optimizer_step(1.0)
    assert log == [("wait", "head"), ("adam", "head"), ("wait", "L1"), ("adam", "L1"), ("wait", "emb"), ("adam", "emb"),
                   ("adam", "L0")]
    assert model._handles == []
