"""Time the GeGLU up-projection GEMM (and a cuBLAS GEMM of the same shape) with whatever library
MB_LIBRARY points to: used with the diagnostic builds of scripts/build_diag.sh."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17482_b200 import _lib

T, Hd, I = 65536, 768, 3072
bf = torch.bfloat16


def timeit(fn, reps=50):
    for _ in range(10):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


torch.manual_seed(0)
X = torch.randn(T, Hd, device="cuda", dtype=bf)
W1v = torch.randn(2 * I, Hd, device="cuda", dtype=bf) * 0.02
b1v = torch.zeros(2 * I, device="cuda", dtype=bf)
Gd = torch.empty(T, 2 * I, device="cuda", dtype=bf)
Z = torch.empty(T, I, device="cuda", dtype=bf)
U = torch.empty(T, 2 * I, device="cuda", dtype=bf)
tag = os.path.basename(os.environ.get("MB_LIBRARY", "") or "tree")
o = timeit(lambda: _lib.geglu_forward(X, W1v, b1v, Gd, Z))
r = timeit(lambda: torch.matmul(X, W1v.t(), out=U))
W2 = torch.randn(Hd, I, device="cuda", dtype=bf) * 0.02
dF = torch.randn(T, Hd, device="cuda", dtype=bf)
dU = torch.empty(T, 2 * I, device="cuda", dtype=bf)
b = timeit(lambda: _lib.geglu_backward(dF, W2, Gd, dU))
print(f"{tag:28s} geglu_fwd {o:7.1f} us ({2*T*2*I*Hd/o/1e6:6.0f} TF/s)  cublas {r:7.1f} us  geglu_bwd {b:7.1f} us", flush=True)
