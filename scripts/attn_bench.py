"""Time the attention forward / backward kernels alone at a config's shape (default C4: 128 x 512,
12 heads, d = 64).  Tuning aid.   usage: attn_bench.py [B] [L]"""
import sys
import numpy as np
import torch
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17482_b200 import _lib as L  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
Lq = int(sys.argv[2]) if len(sys.argv) > 2 else 512
kind = sys.argv[3] if len(sys.argv) > 3 else "full"  # "full" | "lognormal" (the C5 length recipe)
heads, d = 12, 64
H = heads * d
if kind == "full":
    lens = np.full(B, Lq)
else:
    import synth  # noqa: E402
    lens = synth.make_lengths(kind, B, Lq, synth.rng_for(5))
nnz = int(lens.sum())
cu = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)).cuda()
Lq = int(lens.max())
qkv = (torch.randn(nnz, 3 * H, device="cuda") * 0.5).to(torch.bfloat16)
dO = torch.randn(nnz, H, device="cuda").to(torch.bfloat16)
O = torch.empty(nnz, H, dtype=torch.bfloat16, device="cuda")
lse = torch.empty(heads, nnz, device="cuda")
dqkv = torch.empty(nnz, 3 * H, dtype=torch.bfloat16, device="cuda")
db = torch.zeros(3 * H, device="cuda")
sl = torch.from_numpy(L.alibi_slopes(heads)).cuda()
ws = torch.empty(L.attention_workspace_bytes(nnz, heads, d, Lq), dtype=torch.uint8, device="cuda")


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


tf = timed(lambda: L.attention_forward(qkv, cu, B, nnz, Lq, heads, d, sl, O, lse))
tb = timed(lambda: L.attention_backward(qkv, O, dO, lse, cu, B, nnz, Lq, heads, d, sl, dqkv, ws=ws, db_qkv=db))
fl_f = 4.0 * heads * float((lens.astype(np.float64) ** 2).sum()) * d  # QK^T, PV: 2 l^2 d MACs per (seq, head)
fl_b = 2.5 * fl_f                      # S, dP, dV, dK, dQ
byt_f = nnz * (3 * H * 2 + H * 2 + heads * 4)  # QKV in, O + LSE out
print(f"B={B} L={Lq} {kind} nnz={nnz}: attention fwd {tf:.1f} us ({fl_f / tf / 1e6:.0f} TF/s, {byt_f / tf / 1e3:.0f} GB/s), "
      f"bwd (incl. prep/finish) {tb:.1f} us ({fl_b / tb / 1e6:.0f} TF/s)")
