"""Link-prediction ranks (PAPER.md:652-665 [5.3], raw setting) on the CUDA path vs ranks counted
from the oracle's per-triple scores. A candidate whose oracle score lies within fp32 rounding of the true score may
legitimately fall on either side; the allowed rank difference is the number of such near-ties. Both sides score the
same (CUDA-trained) tables."""
import numpy as np
import pytest

import oracle as O
import synth
from paper_2004_08532_b200 import kge

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("model", ["transe_l2", "transe_l1", "distmult", "complex", "rotate"])
@pytest.mark.parametrize("head", [False, True])
def test_ranks_match_oracle(model, head):
    gr = synth.graph("tiny")
    trip = gr.triples()
    cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=32, batch_size=128,
                     chunk_size=32, neg_k=32, gamma=12.0, lr=0.1, seed=2, neg_precision="fp32")
    gpu = kge.init(cfg, *trip)
    orc = O.Trainer(model, gr.n_entities, gr.n_relations, 32, 128, 32, 32, gamma=12.0, lr=0.1, seed=2, triples=trip)
    gpu.train_step(30)
    # ranks are a function of the tables: score the oracle on the CUDA path's trained fp32 rows
    for table, n in ((0, gr.n_entities), (1, gr.n_relations)):
        ids = np.arange(n)
        orc.set_rows(table, ids, gpu.get_rows(table, ids).astype(np.float64))
    rng = np.random.default_rng(11)
    test = rng.integers(0, gr.n_triples, 40)
    hs, rs, ts = trip[0][test], trip[1][test], trip[2][test]
    got = gpu.rank(hs, rs, ts, head=head)
    ents = np.arange(gr.n_entities)
    for i in range(len(test)):
        f_true = orc.score_triples([hs[i]], [rs[i]], [ts[i]])[0]
        if head:
            f = orc.score_triples(ents, np.full_like(ents, rs[i]), np.full_like(ents, ts[i]))
        else:
            f = orc.score_triples(np.full_like(ents, hs[i]), np.full_like(ents, rs[i]), ents)
        ref = 1 + int(np.sum(f > f_true))
        near = int(np.sum(np.abs(f - f_true) <= 1e-4 * (np.abs(f_true) + 1.0)))
        assert abs(int(got[i]) - ref) <= near, (i, got[i], ref, near)
    m = kge.link_metrics(got)
    assert 1.0 <= m["MR"] <= gr.n_entities and 0.0 < m["MRR"] <= 1.0 and m["Hit@1"] <= m["Hit@3"] <= m["Hit@10"]


def test_rank_of_planted_triple_is_one():
    # DistMult with a planted score: make the true tail's row the only one aligned with h * r -> rank 1
    gr = synth.graph("tiny")
    trip = gr.triples()
    cfg = kge.Config(model="distmult", n_entities=gr.n_entities, n_relations=gr.n_relations, dim=8, batch_size=64,
                     chunk_size=16, neg_k=16, neg_precision="fp32")
    gpu = kge.init(cfg, *trip)
    ents = np.arange(gr.n_entities)
    gpu.set_rows(0, ents, np.zeros((gr.n_entities, 8), np.float32))
    gpu.set_rows(0, [3, 7], np.array([[1] * 8, [1] * 8], np.float32))
    gpu.set_rows(1, [0], np.ones((1, 8), np.float32))
    assert gpu.rank([3], [0], [7])[0] == 1  # only e = 3, 7 score > 0; 3 ties 7 exactly (not counted)
    gpu.set_rows(0, [5], np.full((1, 8), 2.0, np.float32))
    assert gpu.rank([3], [0], [7])[0] == 2  # e = 5 now scores higher than the true tail
