"""Link-prediction ranks (PAPER.md:652-665 [5.3]; reading c.15) on the CUDA path vs the oracle's
explicit-sort ranking (oracle.link_rank) on the same tables: raw and filtered first protocol, sampled second protocol.
A candidate whose oracle score lies within fp32 rounding of the positive's may legitimately fall on either side; the
allowed rank difference is the number of such near-ties (0 in almost every query). Both sides score the same
(CUDA-trained) tables."""
import numpy as np
import pytest

import oracle as O
import synth
from paper_2004_08532_b200 import kge

pytestmark = pytest.mark.gpu


def _trained(model, dim=32, steps=30):
    gr = synth.graph("tiny")
    trip = gr.triples()
    cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=dim, batch_size=128,
                     chunk_size=32, neg_k=32, gamma=12.0, lr=0.1, seed=2, neg_precision="fp32")
    gpu = kge.init(cfg, *trip)
    orc = O.Trainer(model, gr.n_entities, gr.n_relations, dim, 128, 32, 32, gamma=12.0, lr=0.1, seed=2, triples=trip)
    gpu.train_step(steps)
    for table, n in ((0, gr.n_entities), (1, gr.n_relations)):
        ids = np.arange(n)
        orc.set_rows(table, ids, gpu.get_rows(table, ids).astype(np.float64))
    return gr, trip, gpu, orc


def _near_ties(orc, n_e, h, r, t, head, cands=None):
    ents = np.arange(n_e) if cands is None else np.asarray(cands, np.int64)
    f_true = orc.score_triples([h], [r], [t])[0]
    if head:
        f = orc.score_triples(ents, np.full_like(ents, r), np.full_like(ents, t))
    else:
        f = orc.score_triples(np.full_like(ents, h), np.full_like(ents, r), ents)
    return int(np.sum(np.abs(f - f_true) <= 1e-4 * (np.abs(f_true) + 1.0)))


@pytest.mark.parametrize("model", ["transe_l2", "transe_l1", "distmult", "complex", "rotate"])
@pytest.mark.parametrize("head", [False, True])
def test_ranks_raw_and_filtered(model, head):
    gr, trip, gpu, orc = _trained(model)
    test = np.random.default_rng(11).integers(0, gr.n_triples, 24)
    hs, rs, ts = trip[0][test], trip[1][test], trip[2][test]
    known = set(zip(*(a.tolist() for a in trip)))
    raw = gpu.rank(hs, rs, ts, head=head)
    fil = gpu.rank(hs, rs, ts, head=head, filters=kge.filter_lists(trip, hs, rs, ts, head=head))
    ref_raw = O.link_rank(orc, hs, rs, ts, head=head)
    ref_fil = O.link_rank(orc, hs, rs, ts, head=head, known=known)
    for i in range(len(test)):
        near = _near_ties(orc, gr.n_entities, hs[i], rs[i], ts[i], head)
        assert abs(int(raw[i]) - int(ref_raw[i])) <= near, (i, raw[i], ref_raw[i], near)
        assert abs(int(fil[i]) - int(ref_fil[i])) <= near, (i, fil[i], ref_fil[i], near)
    assert np.all(fil <= raw)
    m = kge.link_metrics(fil)
    assert 1.0 <= m["MR"] <= gr.n_entities and 0.0 < m["MRR"] <= 1.0 and m["Hit@1"] <= m["Hit@3"] <= m["Hit@10"]


@pytest.mark.parametrize("model", ["transe_l2", "distmult"])
@pytest.mark.parametrize("head", [False, True])
def test_ranks_entity_split(model, head):
    """FB15k-sized entity set: the all-entity kernel splits the entity range over S >= 4 CTAs per query group and adds
    the integer partial counts (split 0 also carries the filter list); 19 queries leave a ragged last group of 3."""
    gr = synth.graph("fb15k")
    trip = gr.triples()
    cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=32, batch_size=128,
                     chunk_size=32, neg_k=32, gamma=12.0, lr=0.1, seed=4, neg_precision="fp32")
    gpu = kge.init(cfg, *trip)
    gpu.train_step(5)
    orc = O.Trainer(model, gr.n_entities, gr.n_relations, 32, 128, 32, 32, gamma=12.0, lr=0.1, seed=4, triples=trip)
    for table, n in ((0, gr.n_entities), (1, gr.n_relations)):
        ids = np.arange(n)
        orc.set_rows(table, ids, gpu.get_rows(table, ids).astype(np.float64))
    test = np.random.default_rng(21).integers(0, gr.n_triples, 19)
    hs, rs, ts = trip[0][test], trip[1][test], trip[2][test]
    filt = kge.filter_lists(trip, hs, rs, ts, head=head)
    known = set()
    for i in range(len(test)):  # the known triples that can occur among these queries' corruptions
        for e in filt[1][filt[0][i]:filt[0][i + 1]]:
            known.add((int(e), int(rs[i]), int(ts[i])) if head else (int(hs[i]), int(rs[i]), int(e)))
    raw = gpu.rank(hs, rs, ts, head=head)
    fil = gpu.rank(hs, rs, ts, head=head, filters=filt)
    ref_raw = O.link_rank(orc, hs, rs, ts, head=head)
    ref_fil = O.link_rank(orc, hs, rs, ts, head=head, known=known)
    for i in range(len(test)):
        near = _near_ties(orc, gr.n_entities, hs[i], rs[i], ts[i], head)
        assert abs(int(raw[i]) - int(ref_raw[i])) <= near, (i, raw[i], ref_raw[i], near)
        assert abs(int(fil[i]) - int(ref_fil[i])) <= near, (i, fil[i], ref_fil[i], near)
    assert np.all(fil <= raw) and np.all(fil >= 1) and np.all(raw <= gr.n_entities)


@pytest.mark.parametrize("model", ["transe_l2", "distmult", "rotate"])
@pytest.mark.parametrize("side", [False, True, "both"])
def test_ranks_sampled_protocol(model, side):
    # second protocol, candidates drawn on the device (reading c.15'); the oracle draws the same counter-based ids
    gr, trip, gpu, orc = _trained(model)
    test = np.random.default_rng(12).integers(0, gr.n_triples, 16)
    hs, rs, ts = trip[0][test], trip[1][test], trip[2][test]
    got = gpu.rank_sampled(hs, rs, ts, head=side, n_uniform=1000, n_degree=1000, seed=3)
    ent, sd = O.eval_candidates(3, gr.n_entities, trip[0], trip[2], len(test), 1000, 1000, both=side == "both")
    if side == "both":
        ref = O.link_rank(orc, hs, rs, ts, head="both", candidates=list(zip(ent, sd)))
    else:
        ref = O.link_rank(orc, hs, rs, ts, head=side, candidates=list(ent))
    for i in range(len(test)):
        near = 0
        for hd in ((False, True) if side == "both" else (side,)):
            c = ent[i][sd[i] == (1 if hd else 0)] if side == "both" else ent[i]
            near += _near_ties(orc, gr.n_entities, hs[i], rs[i], ts[i], hd, c)
        assert abs(int(got[i]) - int(ref[i])) <= near, (i, got[i], ref[i], near)
    assert np.all(got >= 1) and np.all(got <= 2001)


@pytest.mark.parametrize("model", ["transe_l2", "distmult"])
def test_ranks_both_sides_one_list(model):
    # first protocol as PAPER.md:654-655 states it: S_i = the corruptions (h', r, t) and (h, r, t'), raw and filtered
    gr, trip, gpu, orc = _trained(model)
    test = np.random.default_rng(13).integers(0, gr.n_triples, 20)
    hs, rs, ts = trip[0][test], trip[1][test], trip[2][test]
    known = set(zip(*(a.tolist() for a in trip)))
    raw = gpu.rank(hs, rs, ts, head="both")
    fil = gpu.rank(hs, rs, ts, head="both", filters=kge.filter_lists(trip, hs, rs, ts, head="both"))
    ref_raw = O.link_rank(orc, hs, rs, ts, head="both")
    ref_fil = O.link_rank(orc, hs, rs, ts, head="both", known=known)
    for i in range(len(test)):
        near = sum(_near_ties(orc, gr.n_entities, hs[i], rs[i], ts[i], hd) for hd in (False, True))
        assert abs(int(raw[i]) - int(ref_raw[i])) <= near and abs(int(fil[i]) - int(ref_fil[i])) <= near, i
    assert np.all(fil <= raw) and np.all(raw <= 2 * gr.n_entities - 1)


@pytest.mark.parametrize("model", ["transe_l2", "distmult", "complex"])
def test_ranks_production_dim_and_filtered_ties(model):
    # d = 400 (configs[1]/[4]) on the FB15k-sized entity set (entity-split path), plus planted exact ties under a
    # filter: entities whose rows equal the true entity's tie it bit-exactly (pessimistic: they rank above it) unless
    # filtered, in which case they are never scored
    gr = synth.graph("fb15k")
    trip = gr.triples()
    cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=400, batch_size=1024,
                     chunk_size=256, neg_k=256, gamma=12.0, lr=0.1, seed=4, neg_precision="fp32")
    gpu = kge.init(cfg, *trip)
    gpu.train_step(3)
    orc = O.Trainer(model, gr.n_entities, gr.n_relations, 400, 1024, 256, 256, gamma=12.0, lr=0.1, seed=4,
                    triples=trip)
    test = np.random.default_rng(5).integers(0, gr.n_triples, 10)
    hs, rs, ts = trip[0][test], trip[1][test], trip[2][test]
    # plant: copy the true tail's row of query 0 onto 3 other entities; filter 2 of them
    twins = [e for e in (11, 222, 3333) if e not in (int(ts[0]), int(hs[0]))]
    gpu.set_rows(0, twins, np.repeat(gpu.get_rows(0, [ts[0]]), len(twins), 0))
    for table, n in ((0, gr.n_entities), (1, gr.n_relations)):
        ids = np.arange(n)
        orc.set_rows(table, ids, gpu.get_rows(table, ids).astype(np.float64))
    off, ids = kge.filter_lists(trip, hs, rs, ts)
    lists = [list(ids[off[i]:off[i + 1]]) for i in range(len(test))]
    lists[0] += twins[:2]
    off = np.concatenate([[0], np.cumsum([len(x) for x in lists])]).astype(np.int64)
    ids = np.concatenate([np.asarray(x, np.int64) for x in lists])
    fil = gpu.rank(hs, rs, ts, filters=(off, ids))
    raw = gpu.rank(hs, rs, ts)
    known = {(int(hs[i]), int(rs[i]), int(e)) for i in range(len(test)) for e in lists[i]}
    ref_fil = O.link_rank(orc, hs, rs, ts, known=known)
    ref_raw = O.link_rank(orc, hs, rs, ts)
    for i in range(len(test)):
        near = _near_ties(orc, gr.n_entities, hs[i], rs[i], ts[i], False)
        if i == 0:
            near -= len(twins)  # the exact twins are decided exactly (bit-equal scores), not near-ties
        assert abs(int(raw[i]) - int(ref_raw[i])) <= near and abs(int(fil[i]) - int(ref_fil[i])) <= near, (i, raw[i],
                                                                                                           ref_raw[i])
    # the unfiltered twin ties the positive and ranks above it; the filtered ones never count
    assert raw[0] - fil[0] >= 2


def test_rank_planted_and_errors():
    gr = synth.graph("tiny")
    trip = gr.triples()
    cfg = kge.Config(model="distmult", n_entities=gr.n_entities, n_relations=gr.n_relations, dim=8, batch_size=64,
                     chunk_size=16, neg_k=16, neg_precision="fp32")
    gpu = kge.init(cfg, *trip)
    ents = np.arange(gr.n_entities)
    gpu.set_rows(0, ents, np.zeros((gr.n_entities, 8), np.float32))
    gpu.set_rows(0, [3, 7], np.ones((2, 8), np.float32))
    gpu.set_rows(1, [0], np.ones((1, 8), np.float32))
    assert gpu.rank([3], [0], [7])[0] == 2  # e = 3 ties the true tail 7 exactly: pessimistic, it ranks above
    gpu.set_rows(0, [3], np.full((1, 8), 0.5, np.float32))
    assert gpu.rank([3], [0], [7])[0] == 1  # the true tail uniquely maximises
    assert gpu.rank([3], [0], [7], filters=(np.array([0, 1]), np.array([3])))[0] == 1
    assert gpu.rank([3], [0], [7], candidates=(np.array([0, 3]), np.array([7, 7, 5])))[0] == 1
    assert gpu.rank([3], [0], [7], candidates=(np.array([0, 0]), np.zeros(0, np.int64)))[0] == 1  # empty list
    with pytest.raises(kge.KgeError):
        gpu.rank([3], [0], [7], candidates=(np.array([0, 1]), np.array([5])), filters=(np.array([0, 1]), np.array([5])))
    with pytest.raises(kge.KgeError):
        gpu.rank([3], [0], [7], filters=(np.array([0, 1]), np.array([gr.n_entities])))
    with pytest.raises(kge.KgeError):
        gpu.rank([3], [0], [7], candidates=(np.array([1, 0]), np.array([5])))


@pytest.mark.parametrize("model", ["transe_l2", "distmult"])
def test_training_improves_filtered_mrr(model):
    """End-to-end sanity of the training step through the evaluation path: training-triple MRR rises with training.
    The oracle on the same configuration (double) gives filtered MRR 0.0265 -> 0.0865 (TransE-L2) and
    0.0200 -> 0.3217 (DistMult) after 1600 steps; TransE-L2 with gamma = 12 moves slowly (0.0360 after 400 steps)."""
    gr = synth.graph("tiny")
    trip = gr.triples()
    cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=64, batch_size=256,
                     chunk_size=64, neg_k=64, gamma=12.0, lr=0.1, seed=5)
    gpu = kge.init(cfg, *trip)
    test = np.random.default_rng(13).integers(0, gr.n_triples, 200)
    q = (trip[0][test], trip[1][test], trip[2][test])
    filt = kge.filter_lists(trip, *q)
    before = kge.link_metrics(gpu.rank(*q, filters=filt))["MRR"]
    gpu.train_step(1600)
    after = kge.link_metrics(gpu.rank(*q, filters=filt))["MRR"]
    assert after > 2.0 * before, (before, after)


@pytest.mark.parametrize("model", ["transe_l2", "distmult", "complex", "rotate"])
def test_ranks_tcgen05_all_entity(model):
    # on a TF32 handle the all-entity protocol is the tcgen05 contraction S = O E^T (rank_tc.cu). FB15k-sized
    # entity set (117 entity tiles), d = 96, raw / filtered / both sides; against the oracle's explicit-sort ranks with
    # the TF32 near-tie window (candidates whose oracle score lies within 2e-3 (|f_true| + 1) of the positive's may fall
    # on either side), and planted twins of a true entity tie it exactly (pessimistic) unless filtered
    gr = synth.graph("fb15k")
    trip = gr.triples()
    d = 96
    cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=d, batch_size=256,
                     chunk_size=64, neg_k=64, gamma=12.0, lr=0.1, seed=4, neg_precision="tf32")
    gpu = kge.init(cfg, *trip)
    assert gpu.neg_path == "tf32"
    gpu.train_step(5)
    test = np.random.default_rng(8).integers(0, gr.n_triples, 150)  # 2 query tiles, the second ragged
    hs, rs, ts = trip[0][test], trip[1][test], trip[2][test]
    twins = [e for e in (17, 2222, 9999) if e not in (int(ts[0]), int(hs[0]))]
    gpu.set_rows(0, twins, np.repeat(gpu.get_rows(0, [ts[0]]), len(twins), 0))
    orc = O.Trainer(model, gr.n_entities, gr.n_relations, d, 256, 64, 64, gamma=12.0, lr=0.1, seed=4, triples=trip)
    for table, n in ((0, gr.n_entities), (1, gr.n_relations)):
        ids = np.arange(n)
        orc.set_rows(table, ids, gpu.get_rows(table, ids).astype(np.float64))
    off, ids = kge.filter_lists(trip, hs, rs, ts)
    lists = [list(ids[off[i]:off[i + 1]]) for i in range(len(test))]
    lists[0] += twins[:2]
    off = np.concatenate([[0], np.cumsum([len(x) for x in lists])]).astype(np.int64)
    fl = np.concatenate([np.asarray(x, np.int64) for x in lists])
    raw, fil = gpu.rank(hs, rs, ts), gpu.rank(hs, rs, ts, filters=(off, fl))
    known = {(int(hs[i]), int(rs[i]), int(e)) for i in range(len(test)) for e in lists[i]}
    ref_raw, ref_fil = O.link_rank(orc, hs, rs, ts), O.link_rank(orc, hs, rs, ts, known=known)

    def near(i, head=False):
        f_true = orc.score_triples([hs[i]], [rs[i]], [ts[i]])[0]
        ents = np.arange(gr.n_entities)
        f = (orc.score_triples(ents, np.full_like(ents, rs[i]), np.full_like(ents, ts[i])) if head else
             orc.score_triples(np.full_like(ents, hs[i]), np.full_like(ents, rs[i]), ents))
        nt = int(np.sum(np.abs(f - f_true) <= 2e-3 * (abs(f_true) + 1.0)))
        return nt - (len(twins) if (i == 0 and not head) else 0)  # exact twins are decided exactly

    for i in range(len(test)):
        w = near(i)
        assert abs(int(raw[i]) - int(ref_raw[i])) <= w and abs(int(fil[i]) - int(ref_fil[i])) <= w, (i, raw[i], ref_raw[i])
    assert raw[0] - fil[0] >= 2  # the filtered twins never count; the unfiltered one ties and ranks above
    # pooled sides on the tensor-core path: = tail + head - 1 with the one-sided ranks of the same kernel
    both = gpu.rank(hs[:40], rs[:40], ts[:40], head="both")
    assert np.array_equal(both, gpu.rank(hs[:40], rs[:40], ts[:40]) + gpu.rank(hs[:40], rs[:40], ts[:40], head=True) - 1)
