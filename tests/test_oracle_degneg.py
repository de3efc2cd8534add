"""Degree-based in-batch negatives (PAPER.md:437-448 [3.3]): slots j < neg_deg_k of a chunk take
the tail (tail corruption) or head (head corruption) of a uniformly drawn triplet of the mini-batch, so an entity is
drawn with probability proportional to its degree in the mini-batch; the other slots stay uniform."""
import numpy as np

import oracle as O
import synth


def _tr(kd, corrupt=O.ALTERNATE, B=256, g=64, k=64):
    gr = synth.graph("tiny")
    trip = gr.triples()
    return gr, trip, O.Trainer("transe_l2", gr.n_entities, gr.n_relations, 16, B, g, k, seed=7, corrupt=corrupt,
                               triples=trip, neg_deg_k=kd)


def test_zero_mix_is_the_uniform_sampler_and_uniform_slots_unchanged():
    _, _, t0 = _tr(0)
    _, _, t1 = _tr(24)
    for s in (0, 1, 17, 1000):
        p0, n0, m0 = t0.sample(s)
        p1, n1, m1 = t1.sample(s)
        assert np.array_equal(p0, p1) and np.array_equal(m0, m1)
        n0, n1 = n0.reshape(4, 64), n1.reshape(4, 64)
        assert np.array_equal(n0[:, 24:], n1[:, 24:])  # slots j >= k_deg: the c.3 uniform stream, untouched
        assert not np.array_equal(n0[:, :24], n1[:, :24])


def test_in_batch_support_by_mode():
    gr, trip, t = _tr(64)
    h, r, tt = trip
    for s in range(20):
        pos, neg, mode = t.sample(s)
        heads, tails = set(h[pos].tolist()), set(tt[pos].tolist())
        for c in range(4):
            ids = set(neg[c * 64:(c + 1) * 64].tolist())
            assert ids <= (tails if mode[c] == 0 else heads), (s, c)


def test_in_batch_frequency_proportional_to_batch_degree():
    # expected count of entity e over many steps: sum_s k * deg_batch_s(e) / B (tail corruption only)
    gr, trip, t = _tr(64, corrupt=O.TAIL)
    _, _, tt = trip
    obs = np.zeros(gr.n_entities)
    exp = np.zeros(gr.n_entities)
    for s in range(300):
        pos, neg, _ = t.sample(s)
        np.add.at(obs, neg, 1)
        np.add.at(exp, tt[pos], 4 * 64 / 256)
    top = np.argsort(-exp)[:20]  # the hub tails: thousands of draws each
    assert np.all(np.abs(obs[top] - exp[top]) <= 5 * np.sqrt(exp[top]) + 1)
    assert obs.sum() == exp.sum()


def test_training_with_degree_negatives_is_finite():
    _, _, t = _tr(32)
    assert np.all(np.isfinite(t.train(5)))


def test_local_shard_negatives():
    # local negatives: rank w draws uniform negatives from {e : e mod P == w} only; P = 1 unchanged
    gr = synth.graph("tiny")
    trip = gr.triples()
    mk = lambda P, loc: O.Trainer("transe_l2", gr.n_entities, gr.n_relations, 16, 64, 16, 16, seed=7, world_size=P,
                                  triples=trip, neg_local=loc)
    a, b = mk(1, 1), mk(1, 0)
    assert np.array_equal(a.sample(5)[1], b.sample(5)[1])
    for P in (2, 4):
        t = mk(P, 1)
        for w in range(P):
            counts = np.zeros(gr.n_entities)
            for s in range(200):
                _, neg, _ = t.sample(s, w)
                assert np.all(neg % P == w), (P, w)
                np.add.at(counts, neg, 1)
            shard = counts[w::P]
            assert (shard > 0).mean() > 0.9  # covers the shard (12,800 draws over ~1000 / P ids)
