"""The N > 1 plumbing of bench.py / MosaicBert.train_step on one GPU: two ranks under torchrun with
the gloo backend (MB_DIST_BACKEND=gloo; gloo reduces through the host, so no kernel of one rank
waits on the other's).  Checks the data-parallel step end to end — in-stream masked-count
allreduce, per-bucket reductions overlapped with the optimizer, device-side loss normaliser, the
max-over-ranks timing and the JSON line — not its speed (both ranks share the GPU)."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_gloo():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, MB_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--micro", "32", "--accum", "2", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "dp2"
    # 2 ranks x 2 accumulated micro-steps x 32 sequences per optimizer step
    assert line["config"]["global_batch"] == 128 and line["config"]["accumulation"] == 2 and line["value"] > 0
    # the loss is the global mean over both ranks' masked tokens: near ln V at BERT init
    assert 9.0 < line["loss"] < 11.5, line["loss"]
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0


def _dp_worker(rank, world, port, out_dir):
    import numpy as np
    import torch.distributed as dist
    import synth
    import paper_2312_17482_b200 as mb
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = synth.TINY
    params = synth.make_model_params(d, 5, "stress", n_layers=2)
    batch = synth.make_batch("C1", 91, B=8)
    per = 8 // world
    sh = {k: v[rank * per:(rank + 1) * per] for k, v in batch.items()}
    model = mb.MosaicBert(mb.ModelDims(d.hidden, d.heads, d.intermediate, d.vocab, 2, d.ln_eps), params)
    dev = tuple(torch.from_numpy(sh[k]).cuda() for k in ("input_ids", "attention_mask", "labels"))
    loss = model.train_step([dev], optimizer=False)
    torch.cuda.synchronize()
    model.wait_grads()
    n_all = int(((batch["labels"] != -100) & (batch["attention_mask"] != 0)).sum())
    g = model.grads_numpy(scale=1.0 / n_all)
    np.savez(os.path.join(out_dir, f"g{rank}.npz"), loss=float(loss.item()),
             **{f"L{i}_{k}": v for i, lg in enumerate(g["layers"]) for k, v in lg.items()},
             **{k: v for k, v in g.items() if k != "layers"})
    dist.destroy_process_group()


def test_dp_two_ranks_gradient_equals_full_batch(tmp_path):
    """SURVEY §8e invariant with the real kernels: two ranks (gloo, one GPU) on half a batch each,
    gradients summed by the product's bucket allreduce and normalised by the global masked count,
    equal the single-process gradient of the whole batch (fp32 reassociation only)."""
    import numpy as np
    import torch.multiprocessing as mp
    import synth
    import paper_2312_17482_b200 as mb
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mp.start_processes(_dp_worker, args=(2, _port(), str(tmp_path)), nprocs=2, start_method="spawn")
    d = synth.TINY
    params = synth.make_model_params(d, 5, "stress", n_layers=2)
    batch = synth.make_batch("C1", 91, B=8)
    model = mb.MosaicBert(mb.ModelDims(d.hidden, d.heads, d.intermediate, d.vocab, 2, d.ln_eps), params)
    dev = tuple(torch.from_numpy(batch[k]).cuda() for k in ("input_ids", "attention_mask", "labels"))
    loss = float(model.train_step([dev], optimizer=False).item())
    n_all = int(((batch["labels"] != -100) & (batch["attention_mask"] != 0)).sum())
    full = model.grads_numpy(scale=1.0 / n_all)
    r0, r1 = (np.load(tmp_path / f"g{r}.npz") for r in range(2))
    assert abs(float(r0["loss"]) + float(r1["loss"]) - loss) <= 1e-5 * abs(loss)
    for i, lg in enumerate(full["layers"]):
        for k, v in lg.items():
            assert np.array_equal(r0[f"L{i}_{k}"], r1[f"L{i}_{k}"]), k  # both ranks hold the same sum
            scale = max(float(np.abs(v).max()), 1e-30)
            assert float(np.abs(r0[f"L{i}_{k}"] - v).max()) <= 2e-5 * scale, (i, k)
    for k in ("emb", "type_emb", "lne_g", "lne_b", "w_t", "b_t", "lnh_g", "lnh_b", "b_dec"):
        scale = max(float(np.abs(full[k]).max()), 1e-30)
        assert float(np.abs(r0[k] - full[k]).max()) <= 2e-5 * scale, k


def _dp_empty_worker(rank, world, port, out_dir):
    import numpy as np
    import torch.distributed as dist
    import synth
    import paper_2312_17482_b200 as mb
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = synth.TINY
    params = synth.make_model_params(d, 5, "stress", n_layers=2)
    mbs = _empty_case_batches()[rank]
    model = mb.MosaicBert(mb.ModelDims(d.hidden, d.heads, d.intermediate, d.vocab, 2, d.ln_eps), params)
    dev = [tuple(torch.from_numpy(b[k]).cuda() for k in ("input_ids", "attention_mask", "labels")) for b in mbs]
    loss = model.train_step(dev, optimizer=False)
    torch.cuda.synchronize()
    g = model.grads_numpy(scale=float(model.inv_dev.item()))
    np.savez(os.path.join(out_dir, f"e{rank}.npz"), loss=float(loss.item()),
             **{f"L{i}_{k}": v for i, lg in enumerate(g["layers"]) for k, v in lg.items()},
             **{k: v for k, v in g.items() if k != "layers"})
    dist.destroy_process_group()


def _empty_case_batches():
    import numpy as np
    import synth
    a = synth.make_batch("C1", 301, B=4)
    b = synth.make_batch("C1", 302, B=4)
    c = synth.make_batch("C1", 303, B=4)
    empty = {k: v.copy() for k, v in c.items()}
    empty["attention_mask"][:] = 0  # an all-padding micro-batch: nnz == 0
    return [[a, b], [c, empty]]


def test_dp_last_microbatch_all_padding(tmp_path):
    """a rank whose LAST micro-batch is all padding (nnz = 0) must still join the
    masked-count and every bucket allreduce its peer issues (else the job deadlocks), and the
    reduced gradient equals the single-process gradient of all real micro-batches."""
    import time
    import numpy as np
    import torch.multiprocessing as mp
    import synth
    import paper_2312_17482_b200 as mb
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.start_processes(_dp_empty_worker, args=(2, _port(), str(tmp_path)), nprocs=2, start_method="spawn",
                             join=False)
    deadline = time.time() + 300
    while not ctx.join(timeout=5):
        if time.time() > deadline:
            for p in ctx.processes:
                p.kill()
            pytest.fail("data-parallel step with an empty last micro-batch did not finish (deadlock)")
    d = synth.TINY
    params = synth.make_model_params(d, 5, "stress", n_layers=2)
    model = mb.MosaicBert(mb.ModelDims(d.hidden, d.heads, d.intermediate, d.vocab, 2, d.ln_eps), params)
    a, b = _empty_case_batches()[0]
    c, _ = _empty_case_batches()[1]
    dev = [tuple(torch.from_numpy(x[k]).cuda() for k in ("input_ids", "attention_mask", "labels")) for x in (a, b, c)]
    loss = float(model.train_step(dev, optimizer=False).item())
    full = model.grads_numpy(scale=float(model.inv_dev.item()))
    r0, r1 = (np.load(tmp_path / f"e{r}.npz") for r in range(2))
    assert abs(float(r0["loss"]) + float(r1["loss"]) - loss) <= 1e-5 * abs(loss)
    for i, lg in enumerate(full["layers"]):
        for k, v in lg.items():
            assert np.array_equal(r0[f"L{i}_{k}"], r1[f"L{i}_{k}"]), k
            assert float(np.abs(r0[f"L{i}_{k}"] - v).max()) <= 2e-5 * max(float(np.abs(v).max()), 1e-30), (i, k)
    for k in ("emb", "w_t", "b_dec"):
        assert float(np.abs(r0[k] - full[k]).max()) <= 2e-5 * max(float(np.abs(full[k]).max()), 1e-30), k


def _nccl_one_rank_worker(rank, port, out_dir):
    import numpy as np
    import torch.distributed as dist
    import synth
    import paper_2312_17482_b200 as mb
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    opts = dist.ProcessGroupNCCL.Options()
    opts.is_high_priority_stream = True
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0), pg_options=opts)
    d = synth.TINY
    params = synth.make_model_params(d, 7, "stress", n_layers=2)
    dims = mb.ModelDims(d.hidden, d.heads, d.intermediate, d.vocab, 2, d.ln_eps)
    mbs = [synth.make_batch("C1", 400 + i, B=4) for i in range(3)]
    dev = [tuple(torch.from_numpy(b[k]).cuda() for k in ("input_ids", "attention_mask", "labels")) for b in mbs]
    out = {}
    for tag, dp in (("plain", False), ("nccl", True)):
        model = mb.MosaicBert(dims, params)
        if dp:  # one rank, but the whole data-parallel path: count + 14 bucket allreduces through NCCL
            model._dp = lambda: True
        losses = [float(model.train_step(dev).item()) for _ in range(2)]  # two optimizer steps
        torch.cuda.synchronize()
        out[f"{tag}_loss"] = np.array(losses)
        out[f"{tag}_w"] = np.concatenate([b.w.float().cpu().numpy() for b in model.buckets])
    np.savez(os.path.join(out_dir, "nccl1.npz"), **out)
    dist.destroy_process_group()


def test_dp_path_through_nccl_one_rank(tmp_path):
    """The data-parallel step's NCCL data plane on the B200 (one rank: this pool has one GPU): the
    in-stream masked-count allreduce, the 14 per-bucket async allreduces issued during the last
    micro-step's backward on NCCL's high-priority stream, and the optimizer's per-bucket waits.
    Two optimizer steps give bit-identical losses and weights to the non-distributed path (a 1-rank
    sum is exact), so every stream / handle ordering of the NCCL path is exercised end to end."""
    import time
    import numpy as np
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.start_processes(_nccl_one_rank_worker, args=(_port(), str(tmp_path)), nprocs=1, start_method="spawn",
                             join=False)
    deadline = time.time() + 300
    while not ctx.join(timeout=5):
        if time.time() > deadline:
            for p in ctx.processes:
                p.kill()
            pytest.fail("one-rank NCCL data-parallel step did not finish")
    r = np.load(tmp_path / "nccl1.npz")
    assert np.array_equal(r["plain_loss"], r["nccl_loss"]), (r["plain_loss"], r["nccl_loss"])
    assert np.array_equal(r["plain_w"], r["nccl_w"])
