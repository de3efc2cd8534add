"""Whole-step pins for the oracle (Sec. 3.1 four-step loop; readings c.9-c.13):
the oracle's step equals an independent torch.float64 autograd step on the same sampled ids; P ranks equal one
union step with summed losses; float oracle tracks double oracle; training reduces the loss."""
import numpy as np
import pytest
import torch

import oracle as O
from tests import torch_ref as TR

MODELS = ["transe_l1", "transe_l2", "distmult", "complex", "rotate", "transr", "rescal"]


def _tiny_triples(n_e, n_r, n_t, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, n_e, n_t), rng.integers(0, n_r, n_t), rng.integers(0, n_e, n_t)


def _tables(tr, n_e, n_r, has_proj, d):
    E = torch.tensor(tr.get_rows(0, np.arange(n_e)))
    R = torch.tensor(tr.get_rows(1, np.arange(n_r)))
    Pj = torch.tensor(tr.get_rows(2, np.arange(n_r))).view(n_r, d, d) if has_proj else None
    return E, R, Pj


@pytest.mark.parametrize("model", MODELS)
@pytest.mark.parametrize("world", [1, 2])
@pytest.mark.parametrize("loss", ["logistic", "pairwise"])
def test_step_equals_torch_autograd(model, world, loss):
    n_e, n_r, n_t, d, B, g, k = 8, 2, 40, 4, 4, 2, 2
    gamma, lr, eps = 3.0, 0.1, 1e-10
    if loss == "pairwise":  # a margin that leaves some hinges active and some not at these init scales (checked in
        gamma = float(np.float32(0.05))  # tests/test_oracle_ranking_loss.py; the config stores gamma as float)
    variant = 1 if model == "rotate" and world == 2 else 0
    trip = _tiny_triples(n_e, n_r, n_t, 3 + MODELS.index(model))
    tr = O.Trainer(model, n_e, n_r, d, B, g, k, gamma=gamma, lr=lr, eps=eps, seed=11, world_size=world,
                   rotate_variant=variant, triples=trip, loss=loss)
    has_proj = model in ("transr", "rescal")
    E, R, Pj = _tables(tr, n_e, n_r, has_proj, d)
    SE, SR = torch.zeros(n_e, dtype=torch.float64), torch.zeros(n_r, dtype=torch.float64)
    SP = torch.zeros(n_r, dtype=torch.float64)
    for step in range(2):  # two steps: lag-0 ordering (c.12)
        samples = [tr.sample(step, w) for w in range(world)]
        E.requires_grad_(True); R.requires_grad_(True)
        if Pj is not None:
            Pj.requires_grad_(True)
        L = TR.step_loss(model, E, R, Pj, samples, trip, B, g, k, gamma, variant, loss)
        L.backward()
        loss_o = tr.train(1)[0]
        assert abs(loss_o - L.item()) < (1e-12 if step == 0 else 1e-7)
        with torch.no_grad():
            for W, S, in ((E, SE), (R, SR)) + (((Pj, SP),) if Pj is not None else ()):
                G = W.grad
                W.grad = None
                W.requires_grad_(False)
                TR.adagrad_(W, S, G, lr, eps)
        # Adagrad divides by sqrt(mean G^2): gradient sums that cancel to a few ulps (L1 signs) are amplified to
        # ~1e-8 by the different summation order of autograd; a real mistake moves a row by O(lr) = 0.1.
        ATOL = 1e-7
        assert np.allclose(tr.get_rows(0, np.arange(n_e)), E.numpy(), atol=ATOL, rtol=0)
        assert np.allclose(tr.get_rows(1, np.arange(n_r)), R.numpy(), atol=ATOL, rtol=0)
        assert np.allclose(tr.get_rows(3, np.arange(n_e))[:, 0], SE.numpy(), atol=1e-12, rtol=1e-6)
        if has_proj:
            assert np.allclose(tr.get_rows(2, np.arange(n_r)), Pj.reshape(n_r, -1).numpy(), atol=ATOL, rtol=0)


def test_world1_matches_identity_list():
    # P=1 simulation: positives come from the identity list (c.13) -- sample indices are triple indices
    trip = _tiny_triples(50, 5, 100, 1)
    tr = O.Trainer("distmult", 50, 5, 8, 10, 5, 4, seed=2, triples=trip)
    pos, _, _ = tr.sample(0)
    e, r = tr.occurrences(0)
    assert np.array_equal(e[:10], trip[0][pos]) and np.array_equal(r, trip[1][pos])


def test_float_oracle_tracks_double():
    trip = _tiny_triples(200, 10, 2000, 2)
    kw = dict(n_entities=200, n_relations=10, dim=32, batch=64, chunk=16, neg_k=16, gamma=12.0, lr=0.1, seed=4,
              triples=trip)
    td = O.Trainer("transe_l2", precision=0, **kw)
    tf = O.Trainer("transe_l2", precision=1, **kw)
    ld, lf = td.train(20), tf.train(20)
    assert np.allclose(ld, lf, rtol=1e-5)
    ids = np.arange(200)
    assert np.max(np.abs(td.get_rows(0, ids) - tf.get_rows(0, ids))) < 1e-5


@pytest.mark.parametrize("model", MODELS[:5])
def test_training_reduces_loss(model):
    # SPEC.md:438/463 smoke property: loss falls over training on a tiny graph
    trip = _tiny_triples(8, 2, 16, 9)
    tr = O.Trainer(model, 8, 2, 16, 8, 4, 4, gamma=6.0, lr=0.05, seed=3, triples=trip)
    L = tr.train(200)
    assert np.median(L[-20:]) < np.median(L[:20])


def test_lazy_rows_equal_dense():
    trip = _tiny_triples(300, 7, 1000, 5)
    kw = dict(n_entities=300, n_relations=7, dim=16, batch=32, chunk=8, neg_k=8, seed=9, triples=trip)
    a = O.Trainer("complex", **kw)
    b = O.Trainer("complex", lazy_rows=True, **kw)
    assert np.array_equal(a.train(5), b.train(5))
    ids = np.arange(300)
    assert np.array_equal(a.get_rows(0, ids), b.get_rows(0, ids))


def test_generated_graph_callback_equals_arrays():
    import synth
    g = synth.graph("tiny")
    h, r, t = g.triples()
    kw = dict(n_entities=g.n_entities, n_relations=g.n_relations, dim=16, batch=32, chunk=8, neg_k=8, seed=1)
    a = O.Trainer("transe_l2", triples=(h, r, t), **kw)
    b = O.Trainer("transe_l2", graph=g, **kw)
    assert np.array_equal(a.train(3), b.train(3))
