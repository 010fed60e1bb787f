"""MosaicBERT data-parallel training step on the unpadded stream (SURVEY §3 call stack 2).

Host-side orchestration only: every numeric step runs in libmosaicbert.so (see _lib.py).  torch
provides device memory, the CUDA stream and the NCCL process group.

Memory layout (HBM):
  * one flat bf16 parameter buffer and one flat fp32 gradient buffer per encoder layer (the
    layer's allreduce bucket), plus a "head" bucket (MLM transform + LN_h + decoder bias) and an
    "embedding" bucket (E_tok — tied with the decoder, R15 — E_type, LN_e);
  * fp32 master weights + AdamW moments per bucket (F1);
  * per-layer forward "saved" buffers and one backward workspace, sized for the largest micro-batch
    and reused every step (no allocation inside a step).

Data parallelism (P:580 DDP): each rank runs its micro-batches; on the last micro-step
of an optimizer step, each layer's gradient bucket is all-reduced asynchronously as soon as that
layer's backward is enqueued (NCCL orders its stream after the compute stream), so the transfers
overlap the remaining backward.  The loss is the sum over masked tokens divided by the GLOBAL masked
count of the optimizer step (R18), applied as the optimizer's gradient scale.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L

LAYER_SHAPES = lambda H, I: [  # noqa: E731  (nn.Linear W[out, in])
    ("w_qkv", (3 * H, H)), ("b_qkv", (3 * H,)), ("w_o", (H, H)), ("b_o", (H,)), ("ln1_g", (H,)), ("ln1_b", (H,)),
    ("w_1v", (2 * I, H)), ("b_1v", (2 * I,)), ("w_2", (H, I)), ("b_2", (H,)), ("ln2_g", (H,)), ("ln2_b", (H,))]
HEAD_SHAPES = lambda H, V: [("w_t", (H, H)), ("b_t", (H,)), ("lnh_g", (H,)), ("lnh_b", (H,)), ("b_dec", (V,))]  # noqa
EMB_SHAPES = lambda H, V: [("emb", (V, H)), ("type_emb", (2, H)), ("lne_g", (H,)), ("lne_b", (H,))]  # noqa


@dataclasses.dataclass(frozen=True)
class ModelDims:
    hidden: int
    heads: int
    intermediate: int
    vocab: int
    layers: int
    ln_eps: float = 1e-12

    def c(self, deterministic: bool = False) -> L.Dims:
        return L.dims(self.hidden, self.heads, self.intermediate, self.vocab, self.ln_eps, deterministic)


def param_count(d: ModelDims) -> int:
    n = sum(int(np.prod(s)) for _, s in LAYER_SHAPES(d.hidden, d.intermediate)) * d.layers
    n += sum(int(np.prod(s)) for _, s in HEAD_SHAPES(d.hidden, d.vocab))
    n += sum(int(np.prod(s)) for _, s in EMB_SHAPES(d.hidden, d.vocab))
    return n


class Bucket:
    """A flat bf16 parameter buffer + fp32 grad buffer (+ optimizer state) with named views."""

    def __init__(self, shapes, device):
        self.shapes = shapes
        # every view starts 16-byte aligned (TMA / vector loads): offsets rounded up to 8 elements
        self.numel = sum((int(np.prod(s)) + 7) // 8 * 8 for _, s in shapes)
        pad = (self.numel + 63) // 64 * 64
        self.w = torch.zeros(pad, dtype=torch.bfloat16, device=device)
        self.g = torch.zeros(pad, dtype=torch.float32, device=device)
        self.master = None
        self.m = None
        self.v = None
        self.p, self.gv = {}, {}
        o = 0
        for name, s in shapes:
            n = int(np.prod(s))
            self.p[name] = self.w[o:o + n].view(*s)
            self.gv[name] = self.g[o:o + n].view(*s)
            o += (n + 7) // 8 * 8
        self._off = o

    def load(self, src: dict):
        for name, _ in self.shapes:
            v = src[name]
            t = torch.as_tensor(np.asarray(v, dtype=np.float32)) if not torch.is_tensor(v) else v
            self.p[name].copy_(t.to(torch.bfloat16))

    def init_optimizer(self):
        self.master = self.w.float().clone()
        self.m = torch.zeros_like(self.master)
        self.v = torch.zeros_like(self.master)


class MosaicBert:
    """MosaicBERT encoder + MLM head whose forward/backward run in libmosaicbert.so."""

    def __init__(self, dims: ModelDims, params: dict | None = None, device: str | torch.device = "cuda",
                 process_group=None, dropout: float = 0.0, seed: int = 0, lr_peak: float = 5e-4,
                 total_steps: int | None = None, deterministic: bool = False):
        """dropout: F2 feed-forward dropout probability (P:152 uses 0.1; R13/R32).  Each micro-step
        draws its masks from seed_of(micro-step), a pure function of (seed, rank, micro-step index).
        lr_peak / total_steps: the F1 schedule (Table A1: 5e-4 Base, 2e-4 Large).
        deterministic: bitwise-reproducible gradient reductions (MB_FLAG_DETERMINISTIC; slower)."""
        if not 0.0 <= dropout < 1.0:
            raise ValueError("dropout must be in [0, 1)")
        self.dropout = float(dropout)
        self.seed = int(seed)
        self.lr_peak = float(lr_peak)
        self.total_steps = total_steps
        self.micro_index = 0
        self.d = dims
        self.deterministic = bool(deterministic)
        self.cd = dims.c(self.deterministic)
        self.device = torch.device(device)
        L.lib()  # fail loudly now if the library is missing
        H, I, V = dims.hidden, dims.intermediate, dims.vocab
        for name, s in LAYER_SHAPES(H, I):
            assert all(x % 8 == 0 for x in s[-1:]), name
        # bucket offsets must keep every tensor 16-byte aligned: all sizes are multiples of 8
        self.layer_buckets = [Bucket(LAYER_SHAPES(H, I), self.device) for _ in range(dims.layers)]
        self.head_bucket = Bucket(HEAD_SHAPES(H, V), self.device)
        self.emb_bucket = Bucket(EMB_SHAPES(H, V), self.device)
        self.buckets = [*self.layer_buckets, self.head_bucket, self.emb_bucket]
        self.slopes = torch.from_numpy(L.alibi_slopes(dims.heads)).to(self.device)
        self.pg = process_group
        self._cap = (0, 0)
        self._nm_cap = 0
        self.step_count = 0
        self.loss_sum = torch.zeros(1, dtype=torch.float32, device=self.device)
        # R18 on the device: count_dev accumulates n_masked over the micro-steps (mb_mlm_select), is
        # allreduced over the ranks, and mb_loss_normalize turns it into the optimizer's gradient
        # scale (inv_dev) and the returned mean loss (loss_dev) — no host read-back, no torch kernel
        self.count_dev = torch.zeros(1, dtype=torch.float32, device=self.device)
        self.inv_dev = torch.zeros(1, dtype=torch.float32, device=self.device)
        self.loss_dev = torch.zeros(1, dtype=torch.float32, device=self.device)
        self.masked_count = 0
        if params is not None:
            self.load(params)

    # ------------------------------------------------------------------ parameters
    def load(self, params: dict):
        for b, lp in zip(self.layer_buckets, params["layers"]):
            b.load(lp)
        self.head_bucket.load(params)
        self.emb_bucket.load(params)
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)

    def head_params(self):
        h, e = self.head_bucket.p, self.emb_bucket.p
        return L.HeadPtrs(*[L._p(x) for x in (h["w_t"], h["b_t"], h["lnh_g"], h["lnh_b"], e["emb"], h["b_dec"])])

    def head_grads(self):
        h, e = self.head_bucket.gv, self.emb_bucket.gv
        return L.HeadPtrs(*[L._p(x) for x in (h["w_t"], h["b_t"], h["lnh_g"], h["lnh_b"], e["emb"], h["b_dec"])])

    def zero_grad(self):
        for b in self.buckets:
            L.zero_f32(b.g)
        L.zero_f32(self.loss_sum)
        L.zero_f32(self.count_dev)
        self.masked_count = 0

    # ------------------------------------------------------------------ buffers
    def _ensure(self, B: int, Lmax: int):
        if self._cap[0] >= B and self._cap[1] >= Lmax:
            return
        B = max(B, self._cap[0])
        Lmax = max(Lmax, self._cap[1])
        T = B * Lmax
        H = self.d.hidden
        dev = self.device
        self.cu = torch.empty(B + 1, dtype=torch.int32, device=dev)
        self.indices = torch.empty(T, dtype=torch.int32, device=dev)
        self.meta = torch.zeros(4, dtype=torch.int32, device=dev)
        self.idx_ws = torch.empty(max(L.unpad_workspace_bytes(B), 1), dtype=torch.uint8, device=dev)
        self.sel_ws = torch.empty(max(L.select_workspace_bytes(T), 1), dtype=torch.uint8, device=dev)
        self.rows = torch.empty(T, dtype=torch.int32, device=dev)
        self.labs = torch.empty(T, dtype=torch.int32, device=dev)
        self.xs = [torch.empty(T, H, dtype=torch.bfloat16, device=dev) for _ in range(self.d.layers + 1)]
        self.estats = torch.empty(T, 2, dtype=torch.float32, device=dev)
        sb = L.layer_saved_bytes(self.cd, T)
        self.saved = [torch.empty(sb, dtype=torch.uint8, device=dev) for _ in range(self.d.layers)]
        self.ws = torch.empty(L.layer_workspace_bytes(self.cd, T, Lmax), dtype=torch.uint8, device=dev)
        self.dy = [torch.empty(T, H, dtype=torch.bfloat16, device=dev) for _ in range(2)]
        eb = L.embed_workspace_bytes(self.cd, T)
        self.emb_ws = torch.empty(eb, dtype=torch.uint8, device=dev) if eb else None
        self.lse = torch.empty(T, dtype=torch.float32, device=dev)
        self._cap = (B, Lmax)

    def _ensure_head(self, n_m: int):
        if n_m <= self._nm_cap:
            return
        cap = max(n_m, int(self._nm_cap * 1.25) + 64)
        self.head_ws = torch.empty(L.mlm_workspace_bytes(self.cd, cap), dtype=torch.uint8, device=self.device)
        self._nm_cap = cap

    # ------------------------------------------------------------------ one micro-step
    def seed_of(self, micro_index: int) -> int:
        """64-bit dropout seed of one micro-step: a fixed mix of (seed, rank, micro-step index)."""
        rank = dist.get_rank(self.pg) if self._dp() else 0
        x = (self.seed * 0x9E3779B97F4A7C15 + rank * 0xBF58476D1CE4E5B9 + micro_index * 0x94D049BB133111EB)
        return x & 0xFFFFFFFFFFFFFFFF

    @staticmethod
    def batch_meta(mask, labels) -> tuple[int, int, int]:
        """(nnz, max_seqlen, n_masked) of a right-padded batch from HOST arrays (numpy or CPU
        tensors): what mb_unpad_index / mb_mlm_select report, known before the batch is uploaded."""
        m = torch.as_tensor(mask) != 0
        lab = torch.as_tensor(labels)
        return int(m.sum()), int(m.sum(1).max()) if m.numel() else 0, int(((lab != -100) & m).sum())

    def check_meta(self):
        """Verify the device-side index results of the last micro-step run with host_meta against
        the host's numbers (deferred: called at the next micro-step and by train_step's caller at
        its own sync points).  Raises on a mismatch or a device-reported error status."""
        pend = getattr(self, "_meta_pending", None)
        if pend is None:
            return
        self._meta_pending = None
        ev, want, host = pend
        ev.synchronize()
        nnz, max_seqlen, status, n_m = (int(x) for x in host.tolist())
        if status != 0:
            raise RuntimeError(f"batch rejected: {L.STATUS.get(status, status)}")
        if (nnz, max_seqlen, n_m) != tuple(want):
            raise RuntimeError(f"host batch metadata {tuple(want)} != device {(nnz, max_seqlen, n_m)}")

    def micro_step(self, ids: torch.Tensor, mask: torch.Tensor, labels: torch.Tensor, inv_norm: float = 1.0,
                   allreduce: bool = False, timers: dict | None = None, drop_seed: int | None = None,
                   host_meta: tuple[int, int, int] | None = None):
        """Forward + backward of one micro-batch (device int32 [B, L] tensors, right-padded).
        Gradients accumulate (+=) into the buckets.  With dropout, layer l uses mb_dropout(p,
        drop_seed or seed_of(micro-step), stream=l).  Returns (nnz, n_masked)."""
        if drop_seed is None:
            drop_seed = self.seed_of(self.micro_index)
        self.micro_index += 1
        drops = ([L.Dropout(self.dropout, drop_seed, l) for l in range(self.d.layers)] if self.dropout > 0
                 else [None] * self.d.layers)
        B, Lq = mask.shape
        self.check_meta()  # the previous micro-step's deferred check (before _ensure may regrow buffers)
        self._ensure(B, Lq)
        cd = self.cd
        # A1: unpad index (+ token-id range check) + MLM selection; n_masked is also accumulated on
        # the device (count_dev, the R18 normaliser)
        L._ck("mb_unpad_index", L.lib().mb_unpad_index(L._p(mask), L._p(ids), self.d.vocab, B, Lq, L._p(self.cu),
                                                        L._p(self.indices), L._p(self.meta), L._p(self.idx_ws),
                                                        self.idx_ws.numel(), L._stream()))
        L._ck("mb_mlm_select", L.lib().mb_mlm_select(L._p(labels), L._p(self.indices), B * Lq, self.d.vocab,
                                                      L._p(self.rows), L._p(self.labs), L._p(self.meta),
                                                      L._p(self.count_dev), L._p(self.sel_ws), self.sel_ws.numel(),
                                                      L._stream()))
        meta_host = self._meta_host()  # the previous micro-step's copy was consumed by check_meta above
        meta_host.copy_(self.meta, non_blocking=True)
        if host_meta is None:  # read {nnz, max_seqlen, status, n_masked} back (one 16-byte D2H sync)
            torch.cuda.current_stream().synchronize()
            nnz, max_seqlen, status, n_m = (int(x) for x in meta_host.tolist())
            if status != 0:
                raise RuntimeError(f"batch rejected: {L.STATUS.get(status, status)}")
        else:  # sizes known on the host: no sync; the device's numbers are verified later.  They must
            # be exact (batch_meta of the same host arrays): kernels are sized by them
            nnz, max_seqlen, n_m = (int(x) for x in host_meta)
            if not (0 <= n_m <= nnz <= B * Lq and 0 <= max_seqlen <= Lq):
                raise ValueError(f"host_meta {tuple(host_meta)} impossible for a {B}x{Lq} batch")
            ev = torch.cuda.Event()
            ev.record()
            self._meta_pending = (ev, (nnz, max_seqlen, n_m), meta_host)
        self.masked_count += n_m
        if nnz == 0:
            # nothing to compute; a data-parallel rank must still join every collective its peers
            # issue on this micro-step (zero gradients reduce to the right sum)
            if allreduce and self._dp():
                self._count_work = dist.all_reduce(self.count_dev, group=self.pg, async_op=True)
                self._handles = [h for h in (self._allreduce(b) for b in self._reduce_order()) if h is not None]
            return 0, 0
        packed = L.Packed(L._p(self.cu), B, nnz, max_seqlen)
        e = self.emb_bucket.p
        # A3: embedding gather + LN
        L.embed_forward(cd, ids, self.indices, nnz, e["emb"], e["type_emb"], e["lne_g"], e["lne_b"], self.xs[0],
                        self.estats)
        # A4-A9: encoder layers
        lps = [L.layer_ptrs(b.p) for b in self.layer_buckets]
        for l in range(self.d.layers):
            L.encoder_forward(cd, lps[l], packed, self.slopes, self.xs[l], self.xs[l + 1], self.saved[l], drops[l])
        # A11: MLM head + CE (fwd + bwd)
        self._ensure_head(max(n_m, 1))
        dy, dx = self.dy
        t = timers.get("head") if timers else None
        if t is not None:
            t[0].record()
        L.mlm_loss(cd, self.head_params(), self.xs[self.d.layers], nnz, self.rows, self.labs, n_m, inv_norm,
                   self.loss_sum, self.lse, dy, self.head_grads(), self.head_ws)
        if t is not None:
            t[1].record()
        handles = []
        if allreduce and self._dp():
            # the R18 normaliser first (device count of every micro-step so far): its allreduce
            # precedes the gradient buckets in NCCL's order, so the optimizer never waits behind
            # the last bucket; no host value is involved, so nothing synchronises the host
            self._count_work = dist.all_reduce(self.count_dev, group=self.pg, async_op=True)
        if allreduce:
            handles.append(self._allreduce(self.head_bucket))
        # backward through the layers; each bucket's allreduce is issued as soon as it is final
        for l in range(self.d.layers - 1, -1, -1):
            L.encoder_backward(cd, lps[l], packed, self.slopes, self.xs[l], self.saved[l], dy, dx,
                               L.layer_ptrs(self.layer_buckets[l].gv), self.ws, drops[l])
            dy, dx = dx, dy
            if allreduce:
                handles.append(self._allreduce(self.layer_buckets[l]))
        g = self.emb_bucket.gv
        L.embed_backward(cd, ids, self.indices, nnz, e["emb"], e["type_emb"], e["lne_g"], self.estats, dy, g["emb"],
                         g["type_emb"][0], g["lne_g"], g["lne_b"], ws=self.emb_ws)
        if allreduce:
            handles.append(self._allreduce(self.emb_bucket))
        self._handles = [h for h in handles if h is not None]
        return nnz, n_m

    def evaluate(self, ids: torch.Tensor, mask: torch.Tensor, labels: torch.Tensor) -> tuple[float, int]:
        """Forward only, no dropout, no gradients (the inference path of SURVEY F4's "train short,
        test long": ALiBi needs no position table, so the same weights run at any l up to 2048,
        P:131).  Returns (sum over the labelled tokens of their cross-entropy, their count); the
        training state (gradients, the R18 count, the loss accumulator) is left untouched."""
        B, Lq = mask.shape
        self.check_meta()
        self._ensure(B, Lq)
        cd = self.cd
        if getattr(self, "_eval_scalars", None) is None:
            self._eval_scalars = torch.zeros(2, dtype=torch.float32, device=self.device)  # loss, count
        L.zero_f32(self._eval_scalars)
        loss, count = self._eval_scalars[0:1], self._eval_scalars[1:2]
        L._ck("mb_unpad_index", L.lib().mb_unpad_index(L._p(mask), L._p(ids), self.d.vocab, B, Lq, L._p(self.cu),
                                                        L._p(self.indices), L._p(self.meta), L._p(self.idx_ws),
                                                        self.idx_ws.numel(), L._stream()))
        L._ck("mb_mlm_select", L.lib().mb_mlm_select(L._p(labels), L._p(self.indices), B * Lq, self.d.vocab,
                                                      L._p(self.rows), L._p(self.labs), L._p(self.meta),
                                                      L._p(count), L._p(self.sel_ws), self.sel_ws.numel(),
                                                      L._stream()))
        nnz, max_seqlen, status, n_m = (int(x) for x in self.meta.tolist())  # one small D2H read
        if status != 0:
            raise RuntimeError(f"batch rejected: {L.STATUS.get(status, status)}")
        if nnz == 0 or n_m == 0:
            return 0.0, n_m
        packed = L.Packed(L._p(self.cu), B, nnz, max_seqlen)
        e = self.emb_bucket.p
        L.embed_forward(cd, ids, self.indices, nnz, e["emb"], e["type_emb"], e["lne_g"], e["lne_b"], self.xs[0],
                        self.estats)
        for l in range(self.d.layers):
            L.encoder_forward(cd, L.layer_ptrs(self.layer_buckets[l].p), packed, self.slopes, self.xs[l],
                              self.xs[l + 1], self.saved[l], None)
        self._ensure_head(n_m)
        L.mlm_loss(cd, self.head_params(), self.xs[self.d.layers], nnz, self.rows, self.labs, n_m, 1.0, loss,
                   self.lse, None, None, self.head_ws)
        return float(loss.item()), n_m

    def _meta_host(self):
        if getattr(self, "_meta_pinned", None) is None:
            self._meta_pinned = torch.zeros(4, dtype=torch.int32).pin_memory()
        return self._meta_pinned

    def _reduce_order(self):
        """Buckets in the order micro_step issues their allreduce (head, layers L-1..0, embedding)."""
        return [self.head_bucket, *self.layer_buckets[::-1], self.emb_bucket]

    def _dp(self) -> bool:
        return dist.is_available() and dist.is_initialized() and dist.get_world_size(self.pg) > 1

    def _allreduce(self, b: Bucket):
        """Sum one fp32 gradient bucket over the data-parallel ranks (async; A12).  Returns
        (bucket, work) or None."""
        if not self._dp():
            return None
        return b, dist.all_reduce(b.g, op=dist.ReduceOp.SUM, group=self.pg, async_op=True)

    def allreduce_grads(self):
        """Issue the allreduce of every bucket (used when gradients were produced elsewhere)."""
        self._handles = [h for h in (self._allreduce(b) for b in self.buckets) if h is not None]

    def global_masked(self, n_local: int) -> int:
        """N_masked of the whole optimizer step over all ranks (R18: the loss normaliser)."""
        if not self._dp():
            return int(n_local)
        t = torch.tensor([int(n_local)], dtype=torch.int64, device=self.device if self.device.type == "cuda" else "cpu")
        dist.all_reduce(t, group=self.pg)
        return int(t.item())

    def wait_grads(self):
        for _, h in getattr(self, "_handles", []):
            h.wait()
        self._handles = []

    # ------------------------------------------------------------------ optimizer (F1)
    def lr_at(self, step: int) -> float:
        """Warmup + linear decay (Table A1), computed by the library
        (mb_lr_schedule): 0 -> lr_peak over the first 6 % of total_steps, then linearly to
        0.02 lr_peak at total_steps; constant lr_peak if total_steps is None."""
        return L.lr_schedule(step, self.total_steps, self.lr_peak)

    def optimizer_step(self, grad_scale: float, lr: float | None = None, betas=(0.9, 0.98), eps=1e-6,
                       weight_decay: float = 1e-5, grad_scale_dev: torch.Tensor | None = None):
        """Decoupled AdamW (Table A1) over every bucket; rewrites the bf16 weights.  lr
        defaults to the schedule's value at this step; the decay factor handed to the kernel is
        (lr / lr_peak) * weight_decay, not multiplied by lr (reading R34)."""
        self.step_count += 1
        if lr is None:
            lr = self.lr_at(self.step_count)
        wd_step = (lr / self.lr_peak) * weight_decay
        # buckets whose allreduce is still in flight are updated in the order it was issued, each
        # right after its own reduction (stream wait, no host sync): the last bucket's transfer
        # overlaps the other buckets' updates
        pending = getattr(self, "_handles", [])
        self._handles = []
        order = [b for b, _ in pending] + [b for b in self.buckets if all(b is not pb for pb, _ in pending)]
        works = {id(b): w for b, w in pending}
        for b in order:
            if id(b) in works:
                works[id(b)].wait()
            if b.master is None:
                b.init_optimizer()
            L.adamw_step(b.master, b.m, b.v, b.g, b.w, lr, betas[0], betas[1], eps, wd_step, grad_scale,
                         self.step_count, grad_scale_dev=grad_scale_dev)

    # ------------------------------------------------------------------ whole optimizer step
    def train_step(self, micro_batches: Sequence[tuple], global_masked: int | None = None, lr: float | None = None,
                   optimizer: bool = True, host_meta: Sequence[tuple] | None = None):
        """micro_batches: [(ids, mask, labels), ...] device int32 tensors.  Gradients are summed over
        micro-steps (+= contract) and ranks (allreduce on the last micro-step), then scaled by
        1/N_masked_global in the optimizer.  Returns the device loss tensor (mean CE).
        host_meta: optional [batch_meta(mask, labels), ...] computed from the host copy of each
        micro-batch; the step then never waits for the device (its index results are verified one
        micro-step later, check_meta())."""
        self.zero_grad()
        n = len(micro_batches)
        for i, (ids, mask, labels) in enumerate(micro_batches):
            self.micro_step(ids, mask, labels, inv_norm=1.0, allreduce=(i == n - 1),
                            host_meta=host_meta[i] if host_meta is not None else None)
        if global_masked is None and self._dp():
            # R18 normaliser = the global masked count, allreduced in-stream by the last micro-step;
            # mb_loss_normalize turns it into AdamW's device gradient scale and the returned loss
            self._count_work.wait()
            self._count_work = None
            L.loss_normalize(self.loss_sum, count=self.count_dev, inv_out=self.inv_dev, loss_out=self.loss_dev)
            if optimizer:
                self.optimizer_step(1.0, lr=lr, grad_scale_dev=self.inv_dev)  # waits each bucket's reduction
            else:
                self.wait_grads()
            return self.loss_dev
        self.wait_grads()
        if global_masked is None:  # one rank: the device count of this step's micro-steps
            L.loss_normalize(self.loss_sum, count=self.count_dev, inv_out=self.inv_dev, loss_out=self.loss_dev)
        else:
            L.loss_normalize(self.loss_sum, count_host=float(global_masked), inv_out=self.inv_dev,
                             loss_out=self.loss_dev)
        if optimizer:
            self.optimizer_step(1.0, lr=lr, grad_scale_dev=self.inv_dev)
        return self.loss_dev

    def grads_numpy(self, scale: float = 1.0) -> dict:
        """All gradients as float64 numpy arrays in the synth/oracle naming (tests)."""
        out = {"layers": []}
        for b in self.layer_buckets:
            out["layers"].append({k: v.double().cpu().numpy() * scale for k, v in b.gv.items()})
        for b in (self.head_bucket, self.emb_bucket):
            for k, v in b.gv.items():
                out[k] = v.double().cpu().numpy() * scale
        return out
