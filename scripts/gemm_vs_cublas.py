"""Sustained throughput of the library's GEMMs vs cuBLAS (torch.matmul, bf16 out) on the MosaicBERT-Base
layer shapes (65536 tokens).  Tuning aid only; both run back to back in one process."""
import torch
import os, sys  # noqa: E401
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17482_b200 import _lib  # noqa: E402

T, Hd, I = 65536, 768, 3072
dev = "cuda"
bf = torch.bfloat16
torch.manual_seed(0)


def timeit(fn, reps=30):
    for _ in range(5): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def report(name, flops, ours, ref):
    print(f"{name:10s} ours {ours*1e3:8.1f} us {flops/ours/1e9:7.0f} TF/s | cuBLAS {ref*1e3:8.1f} us "
          f"{flops/ref/1e9:7.0f} TF/s | ratio {ref/ours:5.2f}", flush=True)


X = torch.randn(T, Hd, device=dev, dtype=bf)
for name, N, K in (("fwd_qkv", 2304, Hd), ("fwd_o", Hd, Hd), ("fwd_2", Hd, I)):
    A = torch.randn(T, K, device=dev, dtype=bf)
    W = torch.randn(N, K, device=dev, dtype=bf) * 0.02
    C = torch.empty(T, N, device=dev, dtype=bf)
    o = timeit(lambda: _lib.gemm(T, N, K, A, K, 0, W, K, 0, C, N))
    r = timeit(lambda: torch.matmul(A, W.t(), out=C))
    report(name, 2 * T * N * K, o, r)
# out-proj / down-proj as in the layer: + bias + residual (E2)
for name, N, K in (("fwd_o+res", Hd, Hd), ("fwd_2+res", Hd, I)):
    A = torch.randn(T, K, device=dev, dtype=bf)
    W = torch.randn(N, K, device=dev, dtype=bf) * 0.02
    bias = torch.randn(N, device=dev, dtype=bf)
    R = torch.randn(T, N, device=dev, dtype=bf)
    C = torch.empty(T, N, device=dev, dtype=bf)
    o = timeit(lambda: _lib.gemm(T, N, K, A, K, 0, W, K, 0, C, N, bias=bias, residual=R, ldr=N))
    r = timeit(lambda: torch.addmm(bias, A, W.t(), out=C).add_(R))
    report(name, 2 * T * N * K, o, r)
for name, N, K in (("dx_qkv", Hd, 2304), ("dx_1v", Hd, 2 * I), ("dx_o", Hd, Hd)):
    dY = torch.randn(T, K, device=dev, dtype=bf)
    W = torch.randn(K, N, device=dev, dtype=bf) * 0.02
    C = torch.empty(T, N, device=dev, dtype=bf)
    o = timeit(lambda: _lib.gemm(T, N, K, dY, K, 0, W, N, 1, C, N))
    r = timeit(lambda: torch.matmul(dY, W, out=C))
    report(name, 2 * T * N * K, o, r)
for name, M, N in (("dw_qkv", 2304, Hd), ("dw_1v", 2 * I, Hd), ("dw_2", Hd, I), ("dw_o", Hd, Hd)):
    dY = torch.randn(T, M, device=dev, dtype=bf)
    Xn = torch.randn(T, N, device=dev, dtype=bf)
    dW = torch.zeros(M, N, device=dev, dtype=torch.float32)
    Cb = torch.empty(M, N, device=dev, dtype=bf)
    o = timeit(lambda: _lib.gemm_wgrad(M, N, T, dY, M, Xn, N, dW, N))
    r = timeit(lambda: torch.matmul(dY.t(), Xn, out=Cb))
    report(name, 2 * T * N * M, o, r)
W1v = torch.randn(2 * I, Hd, device=dev, dtype=bf) * 0.02
b1v = torch.zeros(2 * I, device=dev, dtype=bf)
Gd = torch.empty(T, 2 * I, device=dev, dtype=bf)
Z = torch.empty(T, I, device=dev, dtype=bf)
U = torch.empty(T, 2 * I, device=dev, dtype=bf)
o = timeit(lambda: _lib.geglu_forward(X, W1v, b1v, Gd, Z))
r = timeit(lambda: torch.matmul(X, W1v.t(), out=U))
report("geglu_fwd", 2 * T * 2 * I * Hd, o, r)
W2 = torch.randn(Hd, I, device=dev, dtype=bf) * 0.02
dF = torch.randn(T, Hd, device=dev, dtype=bf)
dU = torch.empty(T, 2 * I, device=dev, dtype=bf)
dZ = torch.empty(T, I, device=dev, dtype=bf)
o = timeit(lambda: _lib.geglu_backward(dF, W2, Gd, dU))
r = timeit(lambda: torch.matmul(dF, W2, out=dZ))
report("geglu_bwd", 2 * T * I * Hd, o, r)

# mainloop-efficiency probe: the same N with growing K (epilogue cost per FLOP shrinks as K grows)
if __import__("os").environ.get("MB_GEMM_KSWEEP"):
    for N, K in ((2304, 768), (2304, 3072), (2304, 12288), (768, 768), (768, 6144), (4096, 4096)):
        A = torch.randn(T // 4 if K > 4096 else T, K, device=dev, dtype=bf)
        M = A.shape[0]
        W = torch.randn(N, K, device=dev, dtype=bf) * 0.02
        C = torch.empty(M, N, device=dev, dtype=bf)
        o = timeit(lambda: _lib.gemm(M, N, K, A, K, 0, W, K, 0, C, N))
        r = timeit(lambda: torch.matmul(A, W.t(), out=C))
        report(f"k{M}x{N}x{K}", 2 * M * N * K, o, r)
