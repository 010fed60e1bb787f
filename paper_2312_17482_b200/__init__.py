"""B200-native (sm_100a) MosaicBERT data-parallel hot path (arXiv 2312.17482).

The compute lives in ``libmosaicbert.so`` (C ABI declared in ``include/mosaicbert.h``); this package
is the thin Python binding (``_lib``) plus the data-parallel train-step driver (``model``).  The
north_star entry points are re-exported under the paper's names: ``encoder_forward``,
``encoder_backward``, ``mlm_loss``, ``unpad_index``, ``alibi_slopes``.
"""
from ._lib import (  # noqa: F401
    alibi_slopes, attention_backward, attention_forward, colsum, embed_backward, embed_forward, encoder_backward,
    encoder_forward, gather_rows, gemm, geglu_backward, geglu_forward, layernorm_backward, layernorm_forward, lib,
    loss_normalize, mlm_loss, mlm_select, scatter_rows, unpad_index,
)
from .model import ModelDims, MosaicBert, param_count  # noqa: F401

__all__ = ["alibi_slopes", "unpad_index", "mlm_select", "gather_rows", "scatter_rows", "layernorm_forward",
           "layernorm_backward", "gemm", "geglu_forward", "geglu_backward", "attention_forward",
           "attention_backward", "colsum", "encoder_forward", "encoder_backward", "embed_forward",
           "embed_backward", "mlm_loss", "loss_normalize", "ModelDims", "MosaicBert", "param_count", "lib"]
