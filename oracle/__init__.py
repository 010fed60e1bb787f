"""fp64 CPU oracle for the MosaicBERT data-parallel hot path (arXiv 2312.17482).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_2312_17482_b200``) never imports it and shares no code, constants or helpers with it.

It computes the plain PADDED definition in float64 with numpy/scipy, because unpadding and
FlashAttention are exact reformulations of it.  Every function cites the passage it
follows (P:n = PAPER.md line n, S:n = SPEC.md line n; readings R1..R30 are listed in DESIGN.md).

Parity status: every function here is pinned by a ``-m "not gpu"`` test in tests/test_oracle_*.py
(closed forms, worked examples, library special cases, finite differences, an independent torch
fp64 autograd re-implementation).  The whole-model step at full depth (12 and 24 layers) is pinned
by P18 (tests/test_oracle_depth.py): an independent torch-fp64 autograd implementation of the entire
model, loss and every parameter gradient within 1e-9.
"""
from .mosaicbert import *  # noqa: F401,F403
from .mosaicbert import __all__ as _mb_all
from .optim import adamw_step, lr_at  # noqa: F401  (F1, reading R34)

__all__ = [*_mb_all, "adamw_step", "lr_at"]
