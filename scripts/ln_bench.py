"""Time the bf16 LayerNorm forward / backward at C2 size (T = 65536, H = 768).  Tuning aid."""
import torch
import os, sys  # noqa: E401
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17482_b200 import _lib as L  # noqa: E402

import os
T, H = int(os.environ.get("LN_T", 65536)), 768
x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
dy = torch.randn(T, H, device="cuda").to(torch.bfloat16)
g = torch.ones(H, dtype=torch.bfloat16, device="cuda")
b = torch.zeros(H, dtype=torch.bfloat16, device="cuda")
y, dx = torch.empty_like(x), torch.empty_like(x)
st = torch.empty(T, 2, device="cuda")
dg, db, ds = (torch.zeros(H, device="cuda") for _ in range(3))


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


tf = timed(lambda: L.layernorm_forward(x, g, b, 1e-12, y, st))
tb = timed(lambda: L.layernorm_backward(dy, x, st, g, dx, dg, db, ds))
print(f"ln fwd {tf:.1f} us ({2 * T * H * 2 / tf / 1e3:.0f} GB/s)  bwd {tb:.1f} us ({3 * T * H * 2 / tb / 1e3:.0f} GB/s)")
