"""The shared input generator: deterministic, in range, a pure function of (graph_seed, i), shaped per
BASELINE.json configs (Table 3)."""
import numpy as np

import synth


def test_deterministic_and_in_range():
    g = synth.graph("fb15k")
    h, r, t = g.triples(0, 50_000)
    h2, r2, t2 = g.triples(0, 50_000)
    assert np.array_equal(h, h2) and np.array_equal(r, r2) and np.array_equal(t, t2)
    assert h.min() >= 0 and h.max() < g.n_entities and t.max() < g.n_entities
    assert r.min() >= 0 and r.max() < g.n_relations
    # range slices agree with the single-triple function
    for i in (0, 17, 49_999):
        assert g.triple(i) == (h[i], r[i], t[i])
    hh, rr, tt = g.triples(1000, 10, dtype=np.int32)
    assert np.array_equal(hh, h[1000:1010])


def test_skew_and_uniform():
    g = synth.graph("fb15k")
    _, r, _ = g.triples(0, 200_000)
    top = np.bincount(r).max() / len(r)
    assert 0.05 < top < 0.2          # Zipf(1.0) head relation ~ 1/H_N
    gu = synth.graph("fb15k", alpha_e=0.0, alpha_r=0.0)
    _, ru, _ = gu.triples(0, 200_000)
    assert np.bincount(ru).max() / len(ru) < 0.002


def test_freebase_shape_ids_fit_int32():
    g = synth.graph("freebase")
    h, r, t = g.triples(g.n_triples - 1000, 1000)
    assert h.max() < 2 ** 31 and t.max() < g.n_entities
