"""Pins of oracle.embed_forward / embed_backward (A3; "MosaicBERT ... eliminates position
embeddings"; BERT token + token-type embedding + LayerNorm, readings R16/R17/R28).

The oracle is pinned against (i) an independent torch-fp64 re-implementation with library
primitives (F.embedding, F.layer_norm, autograd) and (ii) closed forms that a plausible mistake
breaks: a stray position table (outputs would depend on position), the wrong type row (E_type[1]
instead of E_type[0]), a missing type term, a wrong LN."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O
import synth

pytestmark = pytest.mark.filterwarnings("ignore")


def _case(seed, B=3, L=7, V=50, H=16):
    rng = np.random.default_rng(seed)
    ids = rng.integers(0, V, size=(B, L))
    emb = rng.standard_normal((V, H))
    typ = rng.standard_normal((2, H))
    g = 1.0 + 0.2 * rng.standard_normal(H)
    b = 0.1 * rng.standard_normal(H)
    return ids, emb, typ, g, b


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_embed_forward_matches_torch_fp64(seed):
    ids, emb, typ, g, b = _case(seed)
    eps = 1e-12
    y, _ = O.embed_forward(ids, emb, typ, g, b, eps)
    t = lambda a: torch.tensor(a, dtype=torch.float64)  # noqa: E731
    tok_type = torch.zeros(ids.shape, dtype=torch.long)  # every token has type 0 (R17)
    v = F.embedding(torch.tensor(ids), t(emb)) + F.embedding(tok_type, t(typ))
    ref = F.layer_norm(v, (emb.shape[1],), t(g), t(b), eps)
    assert np.max(np.abs(y - ref.numpy())) <= 1e-12


def test_embed_backward_matches_torch_autograd():
    ids, emb, typ, g, b = _case(7)
    eps = 1e-12
    mask = synth.mask_from_lengths(np.array([7, 4, 1]), 7)
    y, cache = O.embed_forward(ids, emb, typ, g, b, eps)
    R = np.random.default_rng(8).standard_normal(y.shape)
    dE, dT, dg, db = O.embed_backward(R, ids, mask, cache, g, emb.shape[0])
    t = lambda a: torch.tensor(a, dtype=torch.float64, requires_grad=True)  # noqa: E731
    E, T, G, Bb = t(emb), t(typ), t(g), t(b)
    v = F.embedding(torch.tensor(ids), E) + F.embedding(torch.zeros(ids.shape, dtype=torch.long), T)
    out = F.layer_norm(v, (emb.shape[1],), G, Bb, eps)
    (out * torch.tensor(R * mask[..., None])).sum().backward()  # pad positions carry no gradient
    for got, ref in ((dE, E.grad), (dT, T.grad), (dg, G.grad), (db, Bb.grad)):
        assert np.max(np.abs(got - ref.numpy())) <= 1e-10
    assert np.all(dT[1] == 0.0)  # the type-1 row is never used


def test_embed_no_position_dependence():
    """No position table: the output at (b, l) depends on ids[b, l] only — equal ids give
    equal rows at any position, and permuting positions permutes the outputs."""
    ids, emb, typ, g, b = _case(3, B=2, L=9)
    ids[0, 2] = ids[1, 7] = ids[0, 8] = 5
    y, _ = O.embed_forward(ids, emb, typ, g, b)
    assert np.array_equal(y[0, 2], y[1, 7]) and np.array_equal(y[0, 2], y[0, 8])
    perm = np.random.default_rng(0).permutation(9)
    yp, _ = O.embed_forward(ids[:, perm], emb, typ, g, b)
    assert np.array_equal(yp, y[:, perm])


def test_embed_type_row_zero_only():
    """R17: every token has type 0 — E_type[0] enters, E_type[1] never does."""
    ids, emb, typ, g, b = _case(4)
    y, _ = O.embed_forward(ids, emb, typ, g, b)
    t2 = typ.copy()
    t2[1] = 1e6 * np.random.default_rng(1).standard_normal(typ.shape[1])
    assert np.array_equal(O.embed_forward(ids, emb, t2, g, b)[0], y)
    t3 = typ.copy()
    t3[0] += np.linspace(-1, 1, typ.shape[1])
    assert np.max(np.abs(O.embed_forward(ids, emb, t3, g, b)[0] - y)) > 0.1


def test_embed_closed_forms():
    """(a) E_tok[id] + E_type[0] constant along H -> xhat = 0 -> y = beta exactly;
    (b) H = 2, E_tok[id] + E_type[0] = [a, -a] (a >> sqrt(eps)) -> y = [gamma_0 + beta_0, -gamma_1 + beta_1]."""
    V, H = 6, 8
    emb = np.repeat(np.arange(V, dtype=np.float64)[:, None], H, axis=1)  # row i = i * 1
    typ = np.stack([np.full(H, 0.25), np.zeros(H)])
    g, b = np.linspace(0.5, 2.0, H), np.linspace(-1.0, 1.0, H)
    ids = np.array([[0, 3, 5], [1, 1, 2]])
    y, _ = O.embed_forward(ids, emb, typ, g, b, eps=1e-12)
    assert np.array_equal(y, np.broadcast_to(b, y.shape))
    emb2 = np.array([[3.0, -3.0], [0.5, 0.5]])
    typ2 = np.array([[1.0, 1.0], [7.0, -7.0]])  # row 0 of E_tok + E_type[0] = [4, -2] -> xhat = [1, -1]
    g2, b2 = np.array([2.0, 3.0]), np.array([0.5, -0.5])
    y2, _ = O.embed_forward(np.array([[0]]), emb2, typ2, g2, b2, eps=1e-12)
    assert np.allclose(y2[0, 0], [2.0 + 0.5, -3.0 - 0.5], atol=1e-12, rtol=0)
