"""Pins of the oracle's link-prediction ranking (PAPER.md:652-665 [5.3]; reading c.15) and of the host-side evaluation
helpers in kge.py (filter lists, sampled candidate lists, metrics). The ranks are checked against closed-form scores
computed here from the raw tables (DistMult: sum h*r*t; TransE-L2: gamma - ||h + r - t||), not the oracle's scorer."""
import os

import numpy as np
import pytest

import oracle as O
from paper_2004_08532_b200 import kge

GOLD = os.path.join(os.path.dirname(__file__), "golden", "link_metrics_spec.txt")


def _toy(model="distmult", n_e=20, n_r=3, n_t=60, dim=8, seed=0):
    rng = np.random.default_rng(seed)
    trip = tuple(a.astype(np.int64) for a in (rng.integers(0, n_e, n_t), rng.integers(0, n_r, n_t),
                                               rng.integers(0, n_e, n_t)))
    orc = O.Trainer(model, n_e, n_r, dim, 4, 2, 2, gamma=4.0, lr=0.1, seed=1, triples=trip)
    E = rng.normal(size=(n_e, dim))
    R = rng.normal(size=(n_r, dim))
    orc.set_rows(0, np.arange(n_e), E)
    orc.set_rows(1, np.arange(n_r), R)
    return orc, trip, E, R


def _closed_form(model, E, R, h, r, t, gamma=4.0):
    if model == "distmult":
        return float(np.sum(E[h] * R[r] * E[t]))
    return gamma - float(np.linalg.norm(E[h] + R[r] - E[t]))


def test_metrics_golden():
    vals = {ln.split()[0]: ln.split()[1:] for ln in open(GOLD) if ln.strip() and not ln.startswith("#")}
    ranks = [int(x) for x in vals.pop("ranks")]
    for m in (O.link_metrics(ranks), kge.link_metrics(ranks)):
        for k, v in vals.items():
            assert m[k] == pytest.approx(float(v[0]), abs=1e-12), k
    assert O.link_metrics([1, 1, 1]) == {"Hit@1": 1.0, "Hit@3": 1.0, "Hit@10": 1.0, "MR": 1.0, "MRR": 1.0}
    with pytest.raises(ValueError):
        O.link_metrics([])


@pytest.mark.parametrize("model", ["distmult", "transe_l2"])
@pytest.mark.parametrize("head", [False, True])
def test_rank_brute_force_closed_form(model, head):
    orc, trip, E, R = _toy(model)
    q = np.arange(12)
    got = O.link_rank(orc, trip[0][q], trip[1][q], trip[2][q], head=head)
    for i in q:
        h, r, t = int(trip[0][i]), int(trip[1][i]), int(trip[2][i])
        ft = _closed_form(model, E, R, h, r, t)
        sc = [(_closed_form(model, E, R, e, r, t) if head else _closed_form(model, E, R, h, r, e), e)
              for e in range(20) if e != (h if head else t)]
        assert got[i] == 1 + sum(1 for f, _ in sc if f >= ft - 1e-12 * abs(ft)), i


def test_rank_planted_and_all_equal():
    orc, trip, E, R = _toy("distmult")
    h, r, t = int(trip[0][0]), int(trip[1][0]), int(trip[2][0])
    # the positive uniquely maximises the score -> rank 1
    E2 = np.full((20, 8), 0.1)
    E2[t] = 5.0
    E2[h] = 1.0
    orc.set_rows(0, np.arange(20), E2)
    orc.set_rows(1, [r], np.ones((1, 8)))
    assert O.link_rank(orc, [h], [r], [t])[0] == 1
    # all scores equal -> the positive is last among the 20 (pessimistic ties) ...
    orc.set_rows(0, np.arange(20), np.ones((20, 8)))
    assert O.link_rank(orc, [h], [r], [t])[0] == 20
    # ... and filtering removes exactly the known corruptions
    known = set(zip(*(a.tolist() for a in trip)))
    n_known = len({e for (a, b, e) in known if a == h and b == r and e != t})
    assert O.link_rank(orc, [h], [r], [t], known=known)[0] == 20 - n_known


def test_filter_never_worsens_and_order_invariance():
    orc, trip, E, R = _toy("distmult", seed=3)
    q = np.arange(20)
    known = set(zip(*(a.tolist() for a in trip)))
    raw = O.link_rank(orc, trip[0][q], trip[1][q], trip[2][q])
    fil = O.link_rank(orc, trip[0][q], trip[1][q], trip[2][q], known=known)
    assert np.all(fil <= raw) and np.all(fil >= 1)
    orc.set_rows(0, np.arange(20), 3.0 * E)  # scores scale by 9 > 0: a strictly monotone transform
    assert np.array_equal(O.link_rank(orc, trip[0][q], trip[1][q], trip[2][q]), raw)


def test_sampled_protocol_candidates():
    # second protocol (reading c.15'): 1000 uniform + 1000 degree-proportional candidates per query
    orc, trip, E, R = _toy("distmult")
    deg = np.bincount(np.concatenate([trip[0], trip[2]]), minlength=20)
    ent, side = O.eval_candidates(4, 20, trip[0], trip[2], 5, 1000, 1000, both=False)
    assert ent.shape == (5, 2000) and ent.min() >= 0 and ent.max() < 20 and not side.any()  # |S_i| = 2001
    assert not np.any(np.isin(np.nonzero(deg == 0)[0], ent[:, 1000:]))  # degree 0: never drawn
    h, r, t = trip[0][:5], trip[1][:5], trip[2][:5]
    got = O.link_rank(orc, h, r, t, candidates=list(ent))
    for i in range(5):
        ft = _closed_form("distmult", E, R, int(h[i]), int(r[i]), int(t[i]))
        fs = [_closed_form("distmult", E, R, int(h[i]), int(r[i]), int(e)) for e in ent[i] if e != t[i]]
        assert got[i] == 1 + sum(1 for f in fs if f >= ft - 1e-12 * abs(ft))


@pytest.mark.parametrize("both", [False, True])
def test_candidate_draws_uniform_and_degree_proportional(both):
    # 10^6 draws per part: uniform slots are uniform over the entities (both sides pooled: over the (side, entity)
    # pairs); degree slots follow the endpoint degree of the graph ("proportionally to the degree")
    th = np.array([0, 1, 1, 2, 2, 2, 3, 3, 3, 3, 6, 6, 6, 6, 6], np.int64)
    tt = np.array([4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 6, 6, 6, 6, 6], np.int64)
    n_e = 8
    ent, side = O.eval_candidates(9, n_e, th, tt, 1000, 1000, 1000, both=both)
    uni, dg, su, sd = ent[:, :1000].ravel(), ent[:, 1000:].ravel(), side[:, :1000].ravel(), side[:, 1000:].ravel()
    cells = np.bincount(uni * 2 + su if both else uni, minlength=2 * n_e if both else n_e) / len(uni)
    assert np.all(np.abs(cells - cells.mean()) <= 0.02 * cells.mean())
    degree = np.bincount(np.concatenate([th, tt]), minlength=n_e).astype(np.float64)
    freq = np.bincount(dg, minlength=n_e) / len(dg)
    p = degree / degree.sum()
    assert freq[5] == 0 and freq[7] == 0 and np.all(np.abs(freq - p) <= 0.02 * p + 1e-12)
    if both:
        assert abs(sd.mean() - 0.5) < 0.01 and abs(su.mean() - 0.5) < 0.01
    else:
        assert not su.any() and not sd.any()
    # counter-based: the same (seed, query, slot) gives the same draw; another seed does not
    e2, _ = O.eval_candidates(9, n_e, th, tt, 3, 1000, 1000, both=both)
    assert np.array_equal(e2, ent[:3]) and not np.array_equal(O.eval_candidates(10, n_e, th, tt, 3, 1000, 1000,
                                                                                   both=both)[0], ent[:3])


@pytest.mark.parametrize("model", ["distmult", "transe_l2"])
def test_rank_both_sides_one_list(model):
    # S_i holds the corruptions (h', r, t) AND (h, r, t') of the positive; with closed-form scores
    orc, trip, E, R = _toy(model)
    q = np.arange(10)
    known = set(zip(*(a.tolist() for a in trip)))
    for kn in (None, known):
        got = O.link_rank(orc, trip[0][q], trip[1][q], trip[2][q], head="both", known=kn)
        for i in q:
            h, r, t = int(trip[0][i]), int(trip[1][i]), int(trip[2][i])
            ft = _closed_form(model, E, R, h, r, t)
            negs = [(e, r, t) for e in range(20) if e != h] + [(h, r, e) for e in range(20) if e != t]
            if kn is not None:
                negs = [x for x in negs if x not in kn]
            fs = [_closed_form(model, E, R, *x) for x in negs]
            assert got[i] == 1 + sum(1 for f in fs if f >= ft - 1e-12 * abs(ft)), i
        # the pooled list is the union of the two one-sided lists (the positive counted once)
        rt = O.link_rank(orc, trip[0][q], trip[1][q], trip[2][q], head=False, known=kn)
        rh = O.link_rank(orc, trip[0][q], trip[1][q], trip[2][q], head=True, known=kn)
        assert np.array_equal(got, rt + rh - 1)


def test_rank_both_sampled_candidates():
    orc, trip, E, R = _toy("distmult")
    ent, side = O.eval_candidates(2, 20, trip[0], trip[2], 4, 30, 30, both=True)
    h, r, t = trip[0][:4], trip[1][:4], trip[2][:4]
    got = O.link_rank(orc, h, r, t, head="both", candidates=list(zip(ent, side)))
    for i in range(4):
        ft = _closed_form("distmult", E, R, int(h[i]), int(r[i]), int(t[i]))
        fs = [_closed_form("distmult", E, R, int(e), int(r[i]), int(t[i])) if sd else
              _closed_form("distmult", E, R, int(h[i]), int(r[i]), int(e))
              for e, sd in zip(ent[i], side[i]) if e != (h[i] if sd else t[i])]
        assert got[i] == 1 + sum(1 for f in fs if f >= ft - 1e-12 * abs(ft))


def test_filter_lists_match_set():
    rng = np.random.default_rng(7)
    known = tuple(rng.integers(0, 15, 300) for _ in range(3))
    ks = set(zip(*(a.tolist() for a in known)))
    q = rng.integers(0, 300, 40)
    hs, rs, ts = known[0][q], known[1][q], known[2][q]
    for head in (False, True):
        off, ids = kge.filter_lists(known, hs, rs, ts, head=head)
        for i in range(40):
            want = sorted({e for (a, b, c) in ks for e in [a if head else c]
                           if (b == rs[i] and c == ts[i] if head else a == hs[i] and b == rs[i])})
            assert sorted(set(ids[off[i]:off[i + 1]].tolist())) == want


def test_oracle_training_raises_filtered_mrr():
    """The oracle's step descends the logistic loss: a sign error in any score gradient or in the
    Adagrad step would make the training triples' filtered MRR fall instead of rise (DistMult, tiny graph)."""
    import synth
    gr = synth.graph("tiny")
    trip = gr.triples()
    test = np.random.default_rng(13).integers(0, gr.n_triples, 100)
    q = [a[test] for a in trip]
    known = set(zip(*(a.tolist() for a in trip)))
    orc = O.Trainer("distmult", gr.n_entities, gr.n_relations, 64, 256, 64, 64, gamma=12.0, lr=0.1, seed=5,
                    triples=trip)
    before = kge.link_metrics(O.link_rank(orc, *q, known=known))["MRR"]
    losses = orc.train(400)
    after = kge.link_metrics(O.link_rank(orc, *q, known=known))["MRR"]
    assert losses[-50:].mean() < losses[:50].mean()
    assert after > 5.0 * before, (before, after)
