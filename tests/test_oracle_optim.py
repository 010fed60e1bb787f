"""Pins for the F1 oracle (oracle/optim.py): decoupled AdamW (reading R34) and the warmup + linear
decay schedule (Table A1).  CPU only."""
import numpy as np
import pytest
import torch

import oracle as O


def test_adamw_scalar_closed_form():
    """w=1, g=1, t=1, betas (0.9, 0.98), eps 1e-6, lr 0.1, wd 0 -> m_hat = v_hat = 1,
    w' = 1 - 0.1/(1 + 1e-6)."""
    w, m, v = O.adamw_step(np.array([1.0]), np.zeros(1), np.zeros(1), np.array([1.0]), 1, lr=0.1, wd_step=0.0)
    assert m[0] == pytest.approx(0.1, abs=1e-16) and v[0] == pytest.approx(0.02, abs=1e-16)
    assert w[0] == pytest.approx(1.0 - 0.1 / (1.0 + 1e-6), abs=1e-15)


def test_adamw_zero_gradient_and_decoupled_decay():
    """g = 0, wd = 0 -> unchanged; g = 0, decay factor 1e-5 -> w (1 - 1e-5) whatever lr is (R34:
    the decay is not scaled by lr and never passes through Adam's normalisation)."""
    rng = np.random.default_rng(0)
    w0 = rng.standard_normal(64)
    for lr in (1e-4, 5e-4, 1.0):
        w, _, _ = O.adamw_step(w0, np.zeros(64), np.zeros(64), np.zeros(64), 3, lr=lr, wd_step=0.0)
        assert np.array_equal(w, w0)
        w, _, _ = O.adamw_step(w0, np.zeros(64), np.zeros(64), np.zeros(64), 3, lr=lr, wd_step=1e-5)
        assert np.allclose(w, w0 * (1 - 1e-5), rtol=1e-15, atol=0)


def test_adamw_reduces_to_torch_adamw():
    """Library special case: torch.optim.AdamW (fp64) multiplies its decay by lr, so it equals R34
    with wd_step = lr * weight_decay; five steps with a grad_scale, a changing lr and random grads."""
    rng = np.random.default_rng(1)
    n = 257
    w = rng.standard_normal(n)
    p = torch.nn.Parameter(torch.from_numpy(w.copy()))
    opt = torch.optim.AdamW([p], lr=1e-3, betas=(0.9, 0.98), eps=1e-6, weight_decay=0.3)
    m = np.zeros(n)
    v = np.zeros(n)
    for t in range(1, 6):
        g = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 2)
        lr = 1e-3 * t
        for gr in opt.param_groups:
            gr["lr"] = lr
        p.grad = torch.from_numpy(g * 0.25)
        opt.step()
        w, m, v = O.adamw_step(w, m, v, g, t, lr=lr, wd_step=lr * 0.3, grad_scale=0.25)
        assert np.allclose(w, p.detach().numpy(), rtol=1e-13, atol=1e-15), t


def test_lr_schedule_points():
    """Table A1: warmup 6 %, final LR 0.02 LR; linear pieces, continuous at the warmup boundary."""
    T, pk = 70000, 5e-4
    assert O.lr_at(0, T, pk) == 0.0
    assert O.lr_at(4200, T, pk) == pytest.approx(pk, rel=1e-15)
    assert O.lr_at(T, T, pk) == pytest.approx(0.02 * pk, rel=1e-15)
    assert O.lr_at(2100, T, pk) == pytest.approx(0.5 * pk, rel=1e-15)
    assert O.lr_at((4200 + T) // 2, T, pk) == pytest.approx(0.51 * pk, rel=1e-12)
    assert abs(O.lr_at(4201, T, pk) - O.lr_at(4199, T, pk)) < 1e-3 * pk
    with pytest.raises(ValueError):
        O.lr_at(T + 1, T, pk)


def test_model_lr_schedule_matches_oracle():
    """The product's host-side schedule (MosaicBert.lr_at, no GPU needed) equals the oracle's."""
    from paper_2312_17482_b200.model import MosaicBert
    m = MosaicBert.__new__(MosaicBert)
    m.lr_peak, m.total_steps = 2e-4, 1000
    for s in (0, 1, 59, 60, 61, 500, 999, 1000):
        assert m.lr_at(s) == pytest.approx(O.lr_at(s, 1000, 2e-4), rel=1e-12, abs=1e-18)
