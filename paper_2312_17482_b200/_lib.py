"""ctypes binding of libmosaicbert.so — argument marshalling only.

Every function here has the name of the C entry point it wraps (without the ``mb_`` prefix) and
does nothing but turn torch tensors into pointers / sizes and the current CUDA stream into a
``cudaStream_t``; every step of the path runs in the library's kernels.  There is no fallback:
if the library is missing or a call fails, a RuntimeError is raised.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# MB_LIBRARY: an alternative build of the same library (A/B timing of two builds on one box)
LIB_PATH = os.environ.get("MB_LIBRARY") or os.path.join(HERE, "libmosaicbert.so")

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
F32 = C.c_float
SZ = C.c_size_t

EPI_BF16, EPI_F32_ACC, EPI_F32, EPI_GELU_AUX = 0, 1, 2, 3
STATUS = {0: "MB_OK", 1: "MB_ERR_INVALID_ARG", 2: "MB_ERR_CONFIG", 3: "MB_ERR_SHAPE", 4: "MB_ERR_MASK_LAYOUT",
          5: "MB_ERR_LABEL_RANGE", 6: "MB_ERR_WORKSPACE", 7: "MB_ERR_ARCH", 8: "MB_ERR_CUDA",
          9: "MB_ERR_TOKEN_RANGE"}


FLAG_DETERMINISTIC = 1  # mb_dims.flags: bitwise-reproducible gradient reductions


class Dims(C.Structure):
    _fields_ = [("hidden", I32), ("heads", I32), ("intermediate", I32), ("vocab", I32), ("ln_eps", F32),
                ("flags", I32)]


class Packed(C.Structure):
    _fields_ = [("cu_seqlens", P), ("batch", I32), ("nnz", I32), ("max_seqlen", I32)]


class Dropout(C.Structure):
    """mb_dropout (F2, R32): p, seed (one per micro-step and rank), stream (layer index)."""
    _fields_ = [("p", F32), ("seed", C.c_uint64), ("stream", I32)]


LAYER_FIELDS = ("w_qkv", "b_qkv", "w_o", "b_o", "ln1_g", "ln1_b", "w_1v", "b_1v", "w_2", "b_2", "ln2_g", "ln2_b")
HEAD_FIELDS = ("w_t", "b_t", "ln_g", "ln_b", "emb", "b_dec")


class LayerPtrs(C.Structure):
    _fields_ = [(f, P) for f in LAYER_FIELDS]


class HeadPtrs(C.Structure):
    _fields_ = [(f, P) for f in HEAD_FIELDS]


_SIGS = {
    "mb_status_string": (C.c_char_p, [C.c_int]),
    "mb_version": (C.c_char_p, []),
    "mb_launch_count": (C.c_ulonglong, []),
    "mb_probe_set": (C.c_int, [I32, P, I32, P]),
    "mb_alibi_slopes": (C.c_int, [I32, P]),
    "mb_unpad_workspace_bytes": (SZ, [I32]),
    "mb_unpad_index": (C.c_int, [P, P, I32, I32, I32, P, P, P, P, SZ, P]),
    "mb_select_workspace_bytes": (SZ, [I32]),
    "mb_mlm_select": (C.c_int, [P, P, I32, I32, P, P, P, P, P, SZ, P]),
    "mb_loss_normalize": (C.c_int, [P, P, F32, P, P, P]),
    "mb_zero_f32": (C.c_int, [P, C.c_int64, P]),
    "mb_lr_schedule": (C.c_double, [C.c_int64, C.c_int64, C.c_double]),
    "mb_gather_rows": (C.c_int, [P, P, I32, I32, P, P]),
    "mb_scatter_rows": (C.c_int, [P, P, I32, I32, I32, P, P]),
    "mb_layernorm_forward": (C.c_int, [P, P, P, I32, I32, F32, P, P, P]),
    "mb_layernorm_backward": (C.c_int, [P, P, P, P, I32, I32, P, P, P, P, P, P]),
    "mb_gemm": (C.c_int, [I32, I32, I32, P, I64, I32, P, I64, I32, P, I64, I32, P, P, I64, P, I64, P]),
    "mb_gemm_wgrad": (C.c_int, [I32, I32, I32, P, I64, P, I64, P, I64, P, P]),
    "mb_geglu_forward": (C.c_int, [P, I32, I32, I32, P, P, P, P, P]),
    "mb_geglu_backward": (C.c_int, [P, I32, I32, I32, P, P, P, P]),
    "mb_attention_forward": (C.c_int, [P, P, I32, I32, I32, I32, I32, P, P, P, P]),
    "mb_attention_workspace_bytes": (SZ, [I32, I32, I32, I32]),
    "mb_attention_backward": (C.c_int, [P, P, P, P, P, I32, I32, I32, I32, I32, P, P, P, P, SZ, P]),
    "mb_colsum": (C.c_int, [P, I32, I32, P, P]),
    "mb_layer_saved_bytes": (SZ, [C.POINTER(Dims), I32]),
    "mb_layer_workspace_bytes": (SZ, [C.POINTER(Dims), I32, I32]),
    "mb_encoder_forward": (C.c_int, [C.POINTER(Dims), C.POINTER(LayerPtrs), C.POINTER(Packed), P, P, P, P,
                                     C.POINTER(Dropout), P]),
    "mb_encoder_backward": (C.c_int, [C.POINTER(Dims), C.POINTER(LayerPtrs), C.POINTER(Packed), P, P, P, P, P,
                                      C.POINTER(LayerPtrs), P, SZ, C.POINTER(Dropout), P]),
    "mb_dropout_mask": (C.c_int, [C.POINTER(Dropout), I32, I32, I32, P, P]),
    "mb_embed_forward": (C.c_int, [C.POINTER(Dims), P, P, I32, P, P, P, P, P, P, P]),
    "mb_embed_workspace_bytes": (SZ, [C.POINTER(Dims), I32]),
    "mb_embed_backward": (C.c_int, [C.POINTER(Dims), P, P, I32, P, P, P, P, P, P, P, P, P, P, SZ, P]),
    "mb_mlm_workspace_bytes": (SZ, [C.POINTER(Dims), I32]),
    "mb_mlm_loss": (C.c_int, [C.POINTER(Dims), C.POINTER(HeadPtrs), P, I32, P, P, I32, F32, P, P, P,
                              C.POINTER(HeadPtrs), P, SZ, P]),
    "mb_adamw_step": (C.c_int, [P, P, P, P, P, I64, F32, F32, F32, F32, F32, F32, I32, P]),
    "mb_adamw_step_dev": (C.c_int, [P, P, P, P, P, I64, F32, F32, F32, F32, F32, F32, P, I32, P]),
    "mb_layernorm_forward_f32": (C.c_int, [P, P, P, I32, I32, F32, P, P, P]),
    "mb_layernorm_backward_f32": (C.c_int, [P, P, P, P, I32, I32, P, P, P, P, P]),
    "mb_geglu_naive_forward": (C.c_int, [P, P, I64, P, P]),
    "mb_geglu_naive_backward": (C.c_int, [P, P, P, I64, P, P, P]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libmosaicbert.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2312_17482_b200.build`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return sorted(_SIGS)


def _ck(name: str, status: int):
    if status != 0:
        raise RuntimeError(f"{name} failed: {STATUS.get(status, status)}")


def _p(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    assert t.is_cuda and t.is_contiguous(), "device tensors must be contiguous CUDA tensors"
    return t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def launch_count() -> int:
    """Kernels launched by the library in this process so far (host counter)."""
    return int(lib().mb_launch_count())


class Probe:
    """Times every launch of one kernel site inside real steps with CUDA events recorded on the
    launching stream (mb_probe_set).  site: 1 GeGLU GEMM, 2 attention fwd, 3 attention bwd, 4 LN fwd."""

    def __init__(self, site: int, capacity: int = 4096):
        self.site = site
        self.events = [torch.cuda.Event(enable_timing=True) for _ in range(capacity)]
        for e in self.events:  # torch creates the underlying cudaEvent_t lazily, on first record
            e.record()
        torch.cuda.current_stream().synchronize()
        self.handles = (C.c_void_p * capacity)(*[e.cuda_event for e in self.events])
        self.count = C.c_int32(0)
        self.capacity = capacity

    def __enter__(self):
        self.count.value = 0
        _ck("mb_probe_set", lib().mb_probe_set(self.site, self.handles, self.capacity, C.byref(self.count)))
        return self

    def __exit__(self, *a):
        lib().mb_probe_set(0, None, 0, None)

    def times_ms(self):
        n = self.count.value
        return [self.events[2 * i].elapsed_time(self.events[2 * i + 1]) for i in range(n)]


def dims(hidden, heads, intermediate, vocab, ln_eps=1e-12, deterministic=False) -> Dims:
    return Dims(hidden, heads, intermediate, vocab, ln_eps, FLAG_DETERMINISTIC if deterministic else 0)


# --------------------------------------------------------------------------------------- wrappers
def alibi_slopes(heads: int) -> np.ndarray:
    out = np.zeros(max(heads, 1), dtype=np.float32)
    _ck("mb_alibi_slopes", lib().mb_alibi_slopes(heads, out.ctypes.data))
    return out[:heads]


def unpad_workspace_bytes(B: int) -> int:
    return int(lib().mb_unpad_workspace_bytes(B))


def select_workspace_bytes(capacity: int) -> int:
    return int(lib().mb_select_workspace_bytes(capacity))


def _ws(nbytes: int, device, ws):
    """The caller-owned workspace of one call: `ws` if given (must be large enough), else a new one;
    ws=False passes NULL (the single-CTA kernels)."""
    if ws is False or nbytes == 0:
        return None, 0
    if ws is None:
        ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
    return ws, ws.numel()


def unpad_index(mask: torch.Tensor, meta: torch.Tensor | None = None, ids: torch.Tensor | None = None,
                vocab: int = 0, ws=None, out=None):
    """mask: cuda int32 [B, L] -> (cu_seqlens [B+1], indices [B*L] (first nnz valid), meta [4]).
    ids (optional): token ids checked against [0, vocab) (MB_ERR_TOKEN_RANGE in meta[2])."""
    B, L = mask.shape
    if out is None:
        cu = torch.empty(B + 1, dtype=torch.int32, device=mask.device)
        idx = torch.empty(B * L, dtype=torch.int32, device=mask.device)
    else:
        cu, idx = out
    if meta is None:
        meta = torch.zeros(4, dtype=torch.int32, device=mask.device)
    w, nb = _ws(unpad_workspace_bytes(B), mask.device, ws)
    _ck("mb_unpad_index", lib().mb_unpad_index(_p(mask), _p(ids), vocab, B, L, _p(cu), _p(idx), _p(meta), _p(w), nb,
                                               _stream()))
    return cu, idx, meta


def mlm_select(labels: torch.Tensor, indices: torch.Tensor, vocab: int, meta: torch.Tensor, count=None, ws=None,
               out=None):
    cap = indices.numel()
    if out is None:
        rows = torch.empty(cap, dtype=torch.int32, device=labels.device)
        labs = torch.empty(cap, dtype=torch.int32, device=labels.device)
    else:
        rows, labs = out
    w, nb = _ws(select_workspace_bytes(cap), labels.device, ws)
    _ck("mb_mlm_select", lib().mb_mlm_select(_p(labels), _p(indices), cap, vocab, _p(rows), _p(labs), _p(meta),
                                             _p(count), _p(w), nb, _stream()))
    return rows, labs


def loss_normalize(loss_sum, count=None, count_host: float = 0.0, inv_out=None, loss_out=None):
    """R18: inv_out = 1 / max(N, 1), loss_out = loss_sum * inv_out (N from the device `count` or
    count_host)."""
    _ck("mb_loss_normalize", lib().mb_loss_normalize(_p(loss_sum), _p(count), float(count_host), _p(inv_out),
                                                     _p(loss_out), _stream()))


def lr_schedule(step: int, total_steps: int | None, lr_peak: float) -> float:
    """F1 schedule (library host function): warmup 6 %, linear decay to 0.02 lr_peak."""
    return float(lib().mb_lr_schedule(int(step), int(total_steps or 0), float(lr_peak)))


def zero_f32(t):
    """t (fp32 device tensor, contiguous) = 0 through the library (no torch kernel in the step)."""
    _ck("mb_zero_f32", lib().mb_zero_f32(_p(t), t.numel(), _stream()))
    return t


def gather_rows(src, idx, n, dst):
    _ck("mb_gather_rows", lib().mb_gather_rows(_p(src), _p(idx), n, src.shape[-1], _p(dst), _stream()))
    return dst


def scatter_rows(src, idx, n, rows, dst):
    _ck("mb_scatter_rows", lib().mb_scatter_rows(_p(src), _p(idx), n, src.shape[-1], rows, _p(dst), _stream()))
    return dst


def layernorm_forward(x, gamma, beta, eps, y, stats):
    n, H = x.shape
    _ck("mb_layernorm_forward", lib().mb_layernorm_forward(_p(x), _p(gamma), _p(beta), n, H, eps, _p(y), _p(stats),
                                                           _stream()))
    return y, stats


def layernorm_backward(dy, x, stats, gamma, dx, dgamma, dbeta, dsum=None, gelu_pre=None):
    n, H = x.shape
    _ck("mb_layernorm_backward", lib().mb_layernorm_backward(_p(dy), _p(x), _p(stats), _p(gamma), n, H, _p(gelu_pre),
                                                             _p(dx), _p(dgamma), _p(dbeta), _p(dsum), _stream()))
    return dx


def gemm(M, N, K, A, lda, a_t, B, ldb, b_t, Cout, ldc, epilogue=EPI_BF16, bias=None, residual=None, ldr=0, aux=None,
         ldaux=0):
    _ck("mb_gemm", lib().mb_gemm(M, N, K, _p(A), lda, int(a_t), _p(B), ldb, int(b_t), _p(Cout), ldc, epilogue,
                                 _p(bias), _p(residual), ldr, _p(aux), ldaux, _stream()))
    return Cout


def gemm_wgrad(M, N, K, dY, lda, X, ldb, dW, ldc, db=None):
    _ck("mb_gemm_wgrad", lib().mb_gemm_wgrad(M, N, K, _p(dY), lda, _p(X), ldb, _p(dW), ldc, _p(db), _stream()))
    return dW


def geglu_forward(X, w_1v, b_1v, Gd, Z):
    n, H = X.shape
    I = Z.shape[-1]
    _ck("mb_geglu_forward", lib().mb_geglu_forward(_p(X), n, H, I, _p(w_1v), _p(b_1v), _p(Gd), _p(Z), _stream()))
    return Gd, Z


def geglu_backward(dF, w_2, Gd, dU):
    n, H = dF.shape
    I = w_2.shape[1]
    _ck("mb_geglu_backward", lib().mb_geglu_backward(_p(dF), n, H, I, _p(w_2), _p(Gd), _p(dU), _stream()))
    return dU


def attention_forward(qkv, cu_seqlens, batch, nnz, max_seqlen, heads, head_dim, slopes, O, lse):
    _ck("mb_attention_forward", lib().mb_attention_forward(_p(qkv), _p(cu_seqlens), batch, nnz, max_seqlen, heads,
                                                           head_dim, _p(slopes), _p(O), _p(lse), _stream()))
    return O, lse


def attention_workspace_bytes(nnz, heads, head_dim, max_seqlen):
    return int(lib().mb_attention_workspace_bytes(nnz, heads, head_dim, max_seqlen))


def attention_backward(qkv, O, dO, lse, cu_seqlens, batch, nnz, max_seqlen, heads, head_dim, slopes, dqkv, ws=None,
                       db_qkv=None):
    nb = attention_workspace_bytes(nnz, heads, head_dim, max_seqlen)
    if ws is None and nb:
        ws = torch.empty(nb, dtype=torch.uint8, device=qkv.device)
    _ck("mb_attention_backward", lib().mb_attention_backward(_p(qkv), _p(O), _p(dO), _p(lse), _p(cu_seqlens), batch,
                                                             nnz, max_seqlen, heads, head_dim, _p(slopes), _p(dqkv),
                                                             _p(db_qkv), _p(ws), nb, _stream()))
    return dqkv


def colsum(x, out):
    n, Cc = x.shape
    _ck("mb_colsum", lib().mb_colsum(_p(x), n, Cc, _p(out), _stream()))
    return out


def layer_saved_bytes(d: Dims, nnz: int) -> int:
    return int(lib().mb_layer_saved_bytes(C.byref(d), nnz))


def layer_workspace_bytes(d: Dims, nnz: int, max_seqlen: int) -> int:
    return int(lib().mb_layer_workspace_bytes(C.byref(d), nnz, max_seqlen))


def layer_ptrs(p: dict) -> LayerPtrs:
    return LayerPtrs(*[_p(p[f]) for f in LAYER_FIELDS])


def head_ptrs(p: dict) -> HeadPtrs:
    return HeadPtrs(*[_p(p[f]) for f in HEAD_FIELDS])


def _drop(drop):
    return C.byref(drop) if drop is not None else None


def encoder_forward(d: Dims, params, packed: Packed, slopes, x, y, saved, drop: Dropout | None = None):
    lp = params if isinstance(params, LayerPtrs) else layer_ptrs(params)
    _ck("mb_encoder_forward", lib().mb_encoder_forward(C.byref(d), C.byref(lp), C.byref(packed), _p(slopes), _p(x),
                                                       _p(y), _p(saved), _drop(drop), _stream()))
    return y


def encoder_backward(d: Dims, params, packed: Packed, slopes, x, saved, dy, dx, grads, ws,
                     drop: Dropout | None = None):
    lp = params if isinstance(params, LayerPtrs) else layer_ptrs(params)
    lg = grads if isinstance(grads, LayerPtrs) else layer_ptrs(grads)
    _ck("mb_encoder_backward", lib().mb_encoder_backward(C.byref(d), C.byref(lp), C.byref(packed), _p(slopes), _p(x),
                                                         _p(saved), _p(dy), _p(dx), C.byref(lg), _p(ws), ws.numel(),
                                                         _drop(drop), _stream()))
    return dx


def dropout_mask(drop: Dropout, site: int, rows: int, cols: int, out):
    _ck("mb_dropout_mask", lib().mb_dropout_mask(C.byref(drop), site, rows, cols, _p(out), _stream()))
    return out


def embed_forward(d: Dims, ids, indices, nnz, emb, type_emb, ln_g, ln_b, x0, stats):
    _ck("mb_embed_forward", lib().mb_embed_forward(C.byref(d), _p(ids), _p(indices), nnz, _p(emb), _p(type_emb),
                                                   _p(ln_g), _p(ln_b), _p(x0), _p(stats), _stream()))
    return x0


def embed_workspace_bytes(d: Dims, nnz: int) -> int:
    return int(lib().mb_embed_workspace_bytes(C.byref(d), nnz))


def embed_backward(d: Dims, ids, indices, nnz, emb, type_emb, ln_g, stats, dx0, d_emb, d_type_emb, d_ln_g, d_ln_b,
                   ws=None):
    nb = embed_workspace_bytes(d, nnz)
    if ws is None and nb:
        ws = torch.empty(nb, dtype=torch.uint8, device=dx0.device)
    _ck("mb_embed_backward", lib().mb_embed_backward(C.byref(d), _p(ids), _p(indices), nnz, _p(emb), _p(type_emb),
                                                     _p(ln_g), _p(stats), _p(dx0), _p(d_emb), _p(d_type_emb),
                                                     _p(d_ln_g), _p(d_ln_b), _p(ws), ws.numel() if ws is not None else 0,
                                                     _stream()))


def mlm_workspace_bytes(d: Dims, n_masked: int) -> int:
    return int(lib().mb_mlm_workspace_bytes(C.byref(d), n_masked))


def mlm_loss(d: Dims, head, y, nnz, masked_rows, labels, n_masked, inv_norm, loss_sum, lse, dy_top, grads, ws):
    """dy_top = grads = None: forward only (loss_sum += and lse, no gradients)."""
    hp = head if isinstance(head, HeadPtrs) else head_ptrs(head)
    hg = None if grads is None else C.byref(grads if isinstance(grads, HeadPtrs) else head_ptrs(grads))
    _ck("mb_mlm_loss", lib().mb_mlm_loss(C.byref(d), C.byref(hp), _p(y), nnz, _p(masked_rows), _p(labels), n_masked,
                                         inv_norm, _p(loss_sum), _p(lse), _p(dy_top), hg, _p(ws), ws.numel(),
                                         _stream()))


def adamw_step(master, m, v, g, w_bf16, lr, beta1, beta2, eps, weight_decay, grad_scale, step, grad_scale_dev=None):
    if grad_scale_dev is not None:  # device fp32 scalar multiplying grad_scale (no host read-back)
        _ck("mb_adamw_step_dev", lib().mb_adamw_step_dev(_p(master), _p(m), _p(v), _p(g), _p(w_bf16), master.numel(),
                                                         lr, beta1, beta2, eps, weight_decay, grad_scale,
                                                         _p(grad_scale_dev), step, _stream()))
        return
    _ck("mb_adamw_step", lib().mb_adamw_step(_p(master), _p(m), _p(v), _p(g), _p(w_bf16), master.numel(), lr, beta1,
                                             beta2, eps, weight_decay, grad_scale, step, _stream()))


# ---- F3 ablation baselines (not on the training path)
def layernorm_forward_f32(x, gamma, beta, eps, y, stats):
    n, H = x.shape
    _ck("mb_layernorm_forward_f32", lib().mb_layernorm_forward_f32(_p(x), _p(gamma), _p(beta), n, H, eps, _p(y),
                                                                   _p(stats), _stream()))
    return y, stats


def layernorm_backward_f32(dy, x, stats, gamma, dx, dgamma, dbeta, dsum=None):
    n, H = x.shape
    _ck("mb_layernorm_backward_f32", lib().mb_layernorm_backward_f32(_p(dy), _p(x), _p(stats), _p(gamma), n, H, _p(dx),
                                                                     _p(dgamma), _p(dbeta), _p(dsum), _stream()))
    return dx


def geglu_naive_forward(ua, ug, z):
    _ck("mb_geglu_naive_forward", lib().mb_geglu_naive_forward(_p(ua), _p(ug), ua.numel(), _p(z), _stream()))
    return z


def geglu_naive_backward(dz, ua, ug, dua, dug):
    _ck("mb_geglu_naive_backward", lib().mb_geglu_naive_backward(_p(dz), _p(ua), _p(ug), ua.numel(), _p(dua), _p(dug),
                                                                 _stream()))
    return dua, dug
