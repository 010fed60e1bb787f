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
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--micro", "32", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "dp2"
    assert line["config"]["global_batch"] == 64 and line["value"] > 0
    # the loss is the global mean over both ranks' masked tokens: near ln V at BERT init
    assert 9.0 < line["loss"] < 11.5, line["loss"]
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
