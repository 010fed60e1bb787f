"""Time the weight-gradient GEMMs (dW += dY^T X, K = tokens) of one MosaicBERT-Base layer at forced
split-K counts (MB_SPLITK) and with the built-in choice. Tuning aid, not part of the product path."""
import os
import torch
from paper_2312_17482_b200 import _lib

T = 65536
shapes = {"dWqkv": (2304, 768, T), "dWo": (768, 768, T), "dW1v": (6144, 768, T), "dW2": (768, 3072, T),
          "dE": (30528, 768, 19660)}
torch.manual_seed(0)
for name, (M, N, K) in shapes.items():
    dY = torch.randn(K, M, device="cuda", dtype=torch.bfloat16)
    X = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    dW = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    res = []
    for S in [0, 1, 2, 3, 4, 5, 6, 8, 12, 16, 17, 24]:
        if S: os.environ["MB_SPLITK"] = str(S)
        else: os.environ.pop("MB_SPLITK", None)
        for _ in range(3): _lib.gemm_wgrad(M, N, K, dY, M, X, N, dW, N)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(10): _lib.gemm_wgrad(M, N, K, dY, M, X, N, dW, N)
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 100
        res.append(f"{'auto' if S == 0 else S}:{us:.0f}")
    os.environ.pop("MB_SPLITK", None)
    print(f"{name:6s} {2*M*N*K/1e9:6.1f} GF  " + " ".join(res), flush=True)
