"""Library reference point for the attention kernels: torch SDPA (cuDNN and flash backends) on the
same dense shapes scripts/attn_bench.py times with every sequence at full length.  The library runs
WITHOUT the ALiBi bias (an additive mask would add a [B, H, L, L] read), so it does strictly less work
than the MosaicBERT kernels.   usage: attn_vs_cudnn.py B L"""
import sys

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
L = int(sys.argv[2]) if len(sys.argv) > 2 else 512
H, D = 12, 64
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(0)
q, k, v = (torch.randn(B, H, L, D, device=dev, dtype=torch.bfloat16, generator=g).requires_grad_() for _ in range(3))
do = torch.randn(B, H, L, D, device=dev, dtype=torch.bfloat16, generator=g)
flops_f = 4.0 * B * H * L * L * D
flops_b = 2.5 * flops_f


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION)):
    try:
        with sdpa_kernel([be]):
            o = F.scaled_dot_product_attention(q, k, v)
            tf = timed(lambda: F.scaled_dot_product_attention(q, k, v))

            def fb():
                out = F.scaled_dot_product_attention(q, k, v)
                torch.autograd.grad(out, (q, k, v), do)

            tfb = timed(fb)
        tb = tfb - tf
        print(f"[{name}] B={B} L={L}: fwd {tf:.1f} us ({flops_f / tf / 1e6:.0f} TF/s), "
              f"bwd {tb:.1f} us ({flops_b / tb / 1e6:.0f} TF/s)  (no ALiBi)")
    except Exception as e:  # backend not available for this arch / shape
        print(f"[{name}] unavailable: {type(e).__name__}: {str(e).splitlines()[0][:120]}")
