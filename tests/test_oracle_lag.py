"""Oracle lag-1 mode (reading c.12; PAPER.md:515-534 [3.5] "we overlap entity embedding update with the batch
computation in the next mini-batch ... Once the trainer process finishes writing the relation gradients, it proceeds
to the next mini-batch"): step s reads entity rows updated by steps <= s-2, relations by steps <= s-1. Pinned against
the lag-0 oracle with manipulated state, not against itself."""
import numpy as np
import pytest

import oracle as O
import synth

SHAPE = dict(n_dim=16, B=32, g=8, k=8)


def _pair(model, lag):
    gr = synth.graph("tiny")
    trip = gr.triples()
    mk = lambda lg: O.Trainer(model, gr.n_entities, gr.n_relations, SHAPE["n_dim"], SHAPE["B"], SHAPE["g"],
                              SHAPE["k"], gamma=12.0, lr=0.1, seed=3, triples=trip, lag=lg)
    return gr, mk(lag), mk(0)


@pytest.mark.parametrize("model", ["transe_l2", "distmult", "complex", "rotate", "transe_l1"])
def test_first_step_and_relations_match_lag0(model):
    gr, l1, l0 = _pair(model, 1)
    a, b = l1.train(1), l0.train(1)
    assert a[0] == b[0]  # step 0 sees the initial tables either way
    rel = np.arange(gr.n_relations)
    assert np.array_equal(l1.get_rows(1, rel), l0.get_rows(1, rel))  # relations are synchronous
    ent = np.arange(gr.n_entities)
    init = O.Trainer(model, gr.n_entities, gr.n_relations, SHAPE["n_dim"], SHAPE["B"], SHAPE["g"], SHAPE["k"],
                     gamma=12.0, lr=0.1, seed=3, triples=gr.triples())
    assert np.array_equal(l1.get_rows(0, ent), init.get_rows(0, ent))  # entity update of step 0 still held back
    l1.flush()
    assert np.array_equal(l1.get_rows(0, ent), l0.get_rows(0, ent))  # ... and equal to lag 0 once applied
    assert np.array_equal(l1.get_rows(3, ent), l0.get_rows(3, ent))


@pytest.mark.parametrize("model", ["transe_l2", "distmult", "rotate"])
def test_step1_reads_entities_of_step_minus_2(model):
    # lag 1, step 1: relations after step 0, entities initial. Reproduce with lag 0 by undoing step 0's entity update.
    gr, l1, l0 = _pair(model, 1)
    ent = np.arange(gr.n_entities)
    e0, s0 = l0.get_rows(0, ent), l0.get_rows(3, ent)
    l0.train(1)
    l0.set_rows(0, ent, e0)
    l0.set_rows(3, ent, s0)
    a = l1.train(2)
    b = l0.train(1)
    assert a[1] == b[0]


def test_lag1_flush_is_idempotent_and_training_continues():
    gr, l1, l0 = _pair("transe_l2", 1)
    l1.train(3)
    l1.flush()
    ent = np.arange(gr.n_entities)
    x = l1.get_rows(0, ent)
    l1.flush()
    assert np.array_equal(x, l1.get_rows(0, ent))
    assert np.all(np.isfinite(l1.train(2)))
