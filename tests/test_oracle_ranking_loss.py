"""Pins of the oracle's pairwise ranking loss (PAPER.md:247-249 [2]; reading c.9': mean over the B*k (positive,
negative-of-its-chunk) pairs of max(0, gamma - f+ + f-), subgradient 0 at the hinge). Closed forms worked by hand,
the all-active / all-inactive limits, and (tests/test_oracle_step.py) an independent float64 autograd step."""
import numpy as np
import pytest

import oracle as O
from tests import torch_ref as TR  # noqa: F401  (the autograd pin lives in test_oracle_step.py)


def test_hand_worked_example():
    # one positive f+ = 0.5 with negatives f- = [-0.5, 0.2], gamma = 1: margins 1 - 0.5 - 0.5 = 0 (inactive: the
    # hinge at exactly 0 has subgradient 0) and 1 - 0.5 + 0.2 = 0.7 -> L = 0.7 / 2 = 0.35, dL/df- = [0, 1/2],
    # dL/df+ = -1/2
    L, dpos, dneg = O.ranking_loss([0.5], [-0.5, 0.2], 2, 1.0)
    assert L == pytest.approx(0.35, abs=1e-15)
    assert np.allclose(dneg, [0.0, 0.5], atol=0) and np.allclose(dpos, [-0.5], atol=0)


def test_two_positives_rows_pair_with_their_own_negatives():
    # B = 2, k = 2, gamma = 2: positive 0 (f+ = 3) with [0, 2] -> margins [-1, 1]; positive 1 (f+ = -1) with
    # [-4, 0] -> margins [-1, 3]. L = (1 + 3) / 4 = 1; dneg = [0, 1/4, 0, 1/4]; dpos = [-1/4, -1/4]
    L, dpos, dneg = O.ranking_loss([3.0, -1.0], [0.0, 2.0, -4.0, 0.0], 2, 2.0)
    assert L == pytest.approx(1.0, abs=1e-15)
    assert np.array_equal(dneg, [0.0, 0.25, 0.0, 0.25]) and np.array_equal(dpos, [-0.25, -0.25])


def test_limits():
    rng = np.random.default_rng(0)
    B, k = 16, 8
    pos, neg = rng.normal(size=B), rng.normal(size=B * k)
    # every hinge active: L is linear, gamma - mean_i f+_i + mean_ij f-_ij (each positive has k partners)
    L, dpos, dneg = O.ranking_loss(pos, neg, k, 100.0)
    assert L == pytest.approx(100.0 - pos.mean() + neg.mean(), rel=1e-14)
    assert np.allclose(dpos, -1.0 / B) and np.allclose(dneg, 1.0 / (B * k))
    # none active: zero loss and gradients
    L, dpos, dneg = O.ranking_loss(pos, neg, k, -100.0)
    assert L == 0.0 and not dpos.any() and not dneg.any()


def test_inactive_loss_leaves_tables_unchanged():
    # gamma far below every score gap: no active hinge, zero gradients, Adagrad leaves every row as initialised
    rng = np.random.default_rng(1)
    trip = rng.integers(0, 50, 300), rng.integers(0, 4, 300), rng.integers(0, 50, 300)
    tr = O.Trainer("distmult", 50, 4, 8, 16, 4, 4, gamma=-1e6, seed=2, triples=trip, loss="pairwise")
    before = tr.get_rows(0, np.arange(50))
    assert np.all(tr.train(3) == 0.0)
    assert np.array_equal(tr.get_rows(0, np.arange(50)), before)


def test_autograd_config_has_active_and_inactive_hinges():
    # the float64 autograd pin (test_oracle_step.py, gamma = 0.05, seeds 3 + model index) must exercise both sides of
    # the hinge: at step 0 every model but TransE-L2 has active and inactive pairs
    models = ["transe_l1", "transe_l2", "distmult", "complex", "rotate", "transr"]
    mixed = 0
    for mi, model in enumerate(models):
        n_e, n_r, d, B, g, k, gamma = 8, 2, 4, 4, 2, 2, 0.05
        rng = np.random.default_rng(3 + mi)
        trip = rng.integers(0, n_e, 40), rng.integers(0, n_r, 40), rng.integers(0, n_e, 40)
        tr = O.Trainer(model, n_e, n_r, d, B, g, k, gamma=gamma, seed=11, triples=trip, loss="pairwise")
        pos, neg, mode = tr.sample(0)
        h, r, t = (a[pos] for a in trip)
        fpos = tr.score_triples(h, r, t)
        negs = neg.reshape(len(mode), k)
        m = []
        for i in range(B):
            c = i // g
            hh = np.full(k, h[i]) if mode[c] == 0 else negs[c]
            tt = negs[c] if mode[c] == 0 else np.full(k, t[i])
            m.append(gamma - fpos[i] + tr.score_triples(hh, np.full(k, r[i]), tt))
        m = np.concatenate(m)
        mixed += int((m > 0).any() and (m <= 0).any())
    assert mixed >= 5, mixed
