"""P > 1 ranks on one GPU (single-process emulation: P handles, one stream each, connected directly) against the
oracle's P-rank simulation (reading c.13: one step over the union of the rank batches, losses summed; entity gradients
summed at the owner before one Adagrad step; split relations summed in rank order). The kernels are the multi-process
ones: rows are read through the owner's shard pointer, owners pull gradients, device barriers order the phases."""
import numpy as np
import pytest

import oracle as O
import synth
from paper_2004_08532_b200 import kge

pytestmark = pytest.mark.gpu


def _run(model, P, shape, steps, precision="fp32", graph="tiny", variant=0, neg_local=0, neg_deg_k=0, lag=0,
         repartition=0):
    B, g, k, d = shape
    gr = synth.graph(graph)
    trip = gr.triples()
    cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=d, batch_size=B,
                     chunk_size=g, neg_k=k, neg_precision=precision, rotate_variant=variant, neg_local=neg_local,
                     neg_deg_k=neg_deg_k, lag=lag, repartition=repartition)
    hs = kge.init_local_group(cfg, P, *trip)
    orc = O.Trainer(model, gr.n_entities, gr.n_relations, d, B, g, k, world_size=P, triples=trip,
                    rotate_variant=variant, neg_local=neg_local, neg_deg_k=neg_deg_k, lag=lag, repartition=repartition)
    # integer half per rank: bit-exact
    for w in range(P):
        s = hs[w].sample(3)
        pos, neg, mode = orc.sample(3, w)
        assert np.array_equal(s["pos"], pos) and np.array_equal(s["neg"], neg) and np.array_equal(s["mode"], mode)
    for _ in range(steps):
        for h in hs:
            h.train_step(1, return_loss=False)
    for h in hs:
        h.sync()
    lg = sum(h.read_losses(0, steps).astype(np.float64) for h in hs)
    lo = orc.train(steps)
    return gr, hs, orc, lg, lo


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("model", ["transe_l2", "distmult", "rotate"])
def test_dist_parity_fp32(model, P):
    gr, hs, orc, lg, lo = _run(model, P, (128, 32, 32, 32), 30)
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= 1e-5, (lg[:5], lo[:5])
    ids = np.arange(gr.n_entities)
    got = np.stack([hs[e % P].get_rows(0, [e])[0] for e in ids])
    assert np.abs(got - orc.get_rows(0, ids)).max() <= 1e-4
    rids = np.arange(gr.n_relations)
    owners = [hs[0].relation_owner(r) for r in rids]
    rel = np.stack([hs[max(o, 0)].get_rows(1, [r])[0] for r, o in zip(rids, owners)])
    assert np.abs(rel - orc.get_rows(1, rids)).max() <= 1e-4
    st = np.stack([hs[e % P].get_rows(3, [e])[0] for e in ids])
    assert np.abs(st[:, 0] - orc.get_rows(3, ids)[:, 0]).max() <= 1e-6


def test_dist_split_relations_and_tf32():
    # tiny has 20 Zipf relations: at P = 8 the heavy ones exceed N_t/P and are split (replicated, summed in rank order)
    gr, hs, orc, lg, lo = _run("transe_l2", 8, (256, 64, 64, 64), 20, precision="tf32")
    assert any(hs[0].relation_owner(r) == -1 for r in range(gr.n_relations))
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= 2e-3
    # split relation replicas agree exactly on every rank
    for r in range(gr.n_relations):
        if hs[0].relation_owner(r) == -1:
            rows = [h.get_rows(1, [r]) for h in hs]
            assert all(np.array_equal(rows[0], x) for x in rows[1:])


def test_dist_requires_connect_and_owner_rows():
    gr = synth.graph("tiny")
    trip = gr.triples()
    cfg = kge.Config(model="transe_l2", n_entities=gr.n_entities, n_relations=gr.n_relations, dim=32, batch_size=64,
                     chunk_size=16, neg_k=16, world_size=2, rank=1)
    h = kge.init(cfg, *trip)
    with pytest.raises(kge.KgeError) as ei:
        h.train_step(1)
    assert ei.value.status == -7
    with pytest.raises(kge.KgeError):
        h.get_rows(0, [0])  # entity 0 is owned by rank 0
    assert h.get_rows(0, [1]).shape == (1, 32)


@pytest.mark.parametrize("P", [2, 4])
def test_dist_local_and_degree_negatives(P):
    # local-shard negatives + degree-based in-batch slots on the P-rank path
    gr, hs, orc, lg, lo = _run("transe_l2", P, (128, 32, 32, 32), 20, neg_local=1, neg_deg_k=8)
    for w in range(P):
        assert np.all(hs[w].sample(4)["neg"].reshape(4, 32)[:, 8:] % P == w)
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= 1e-5
    ids = np.arange(gr.n_entities)
    got = np.stack([hs[e % P].get_rows(0, [e])[0] for e in ids])
    assert np.abs(got - orc.get_rows(0, ids)).max() <= 1e-4


@pytest.mark.parametrize("P,precision", [(2, "fp32"), (4, "fp32"), (8, "fp32"), (4, "tf32")])
def test_dist_transr_relation_partitioned(P, precision):
    # configs[3]: TransR relation-partitioned across P ranks (M_r of a relation lives and is
    # updated on its owner only; split relations' M_r replicated, rank sums exchanged). Union-batch semantics of
    # reading c.13 against the oracle's P-rank simulation.
    gr, hs, orc, lg, lo = _run("transr", P, (128, 32, 32, 16), 12, precision=precision)
    tol = 1e-5 if precision == "fp32" else 2e-3
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= tol, (lg[:4], lo[:4])
    ids, rids = np.arange(gr.n_entities), np.arange(gr.n_relations)
    got = np.stack([hs[e % P].get_rows(0, [e])[0] for e in ids])
    rtol = 1e-4 if precision == "fp32" else 2e-2
    assert np.abs(got - orc.get_rows(0, ids)).max() <= rtol
    owners = [hs[0].relation_owner(r) for r in rids]
    for tab in (1, 2, 5):  # relation rows, projections M_r, projection Adagrad states: from the owner (or any replica)
        mine = np.stack([hs[max(o, 0)].get_rows(tab, [r])[0] for r, o in zip(rids, owners)])
        ref = orc.get_rows(tab, rids)
        stol = (1e-6 if precision == "fp32" else 2e-3 * np.abs(ref).max()) if tab == 5 else rtol
        assert np.abs(mine - ref).max() <= stol, tab
    if P == 8:
        split = [r for r, o in zip(rids, owners) if o == -1]
        assert split, "P = 8 must split the heavy relations of the tiny graph"
        for r in split:  # replicas agree exactly
            rows = [h.get_rows(2, [r]) for h in hs]
            assert all(np.array_equal(rows[0], x) for x in rows[1:])


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("model,precision", [("transe_l2", "fp32"), ("distmult", "fp32"), ("transe_l2", "tf32")])
def test_dist_lag1_overlapped_owner_update(model, precision, P):
    # lag = 1 at P > 1 (reading c.12; PAPER.md:515-534 the entity update overlaps the next mini-batch; north_star: the
    # gradient return "overlapped with the next batch's compute"): the owner update of step s runs on the update stream
    # while step s+1 computes, after every rank's step-s+1 entity reads. Oracle: the same lag-1 order at P ranks.
    gr, hs, orc, lg, lo = _run(model, P, (128, 32, 32, 32), 25, precision=precision, lag=1)
    tol = 1e-5 if precision == "fp32" else 2e-3
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= tol, (lg[:4], lo[:4])
    # entity rows: the last step's owner update is held back; reading them first needs the collective flush
    with pytest.raises(kge.KgeError) as ei:
        hs[0].get_rows(0, [0])
    assert ei.value.status == -7
    rids = np.arange(gr.n_relations)  # relations are synchronous: readable now
    owners = [hs[0].relation_owner(r) for r in rids]
    rel = np.stack([hs[max(o, 0)].get_rows(1, [r])[0] for r, o in zip(rids, owners)])
    rtol = 1e-4 if precision == "fp32" else 2e-2
    assert np.abs(rel - orc.get_rows(1, rids)).max() <= rtol
    for h in hs:
        h.flush()
    orc.flush()
    ids = np.arange(gr.n_entities)
    got = np.stack([hs[e % P].get_rows(0, [e])[0] for e in ids])
    assert np.abs(got - orc.get_rows(0, ids)).max() <= rtol
    st = np.stack([hs[e % P].get_rows(3, [e])[0] for e in ids])
    assert np.abs(st[:, 0] - orc.get_rows(3, ids)[:, 0]).max() <= (1e-6 if precision == "fp32" else 1e-3)
    # and it really is the lag-1 trajectory, not lag 0
    _, _, _, lg0, _ = _run(model, P, (128, 32, 32, 32), 5, precision=precision, lag=0)
    assert lg[0] == pytest.approx(lg0[0], rel=1e-6) and np.any(np.abs(lg[2:5] - lg0[2:5]) > 1e-7)


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("model", ["transe_l2", "transr"])
def test_dist_epoch_repartition(model, P):
    # per-epoch randomised relation repartition (reading c.13'): the tiny graph at B = 128 has
    # S_E = ceil(10000 / (P 128)) = 40 / 20 steps per epoch, so 1 / 2 epoch switches happen in the 60-step run (the
    # loss ring keeps 64 steps); positives bit-exact per rank and step, losses and tables vs the oracle's P-rank
    # simulation with the same per-epoch partitions
    d = 16 if model == "transr" else 32
    steps = 60
    gr, hs, orc, lg, lo = _run(model, P, (128, 32, 32, d), steps, repartition=1)
    SE = -(-gr.n_triples // (P * 128))
    assert steps > SE
    for w in range(P):  # sampling bit-exact in the last epoch
        s = hs[w].sample(steps - 1)
        assert np.array_equal(s["pos"], orc.sample(steps - 1, w)[0])
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= 1e-5, (lg[:4], lo[:4])
    ids, rids = np.arange(gr.n_entities), np.arange(gr.n_relations)
    got = np.stack([hs[e % P].get_rows(0, [e])[0] for e in ids])
    assert np.abs(got - orc.get_rows(0, ids)).max() <= 1e-4
    # relation rows: the current epoch's owner (or any replica of a split relation) holds the oracle's row
    owners = [hs[0].relation_owner(r) for r in rids]
    rel = np.stack([hs[max(o, 0)].get_rows(1, [r])[0] for r, o in zip(rids, owners)])
    assert np.abs(rel - orc.get_rows(1, rids)).max() <= 1e-4
    e_now = (steps - 1) // SE
    o_now, _ = O.relation_partition(gr.triples()[1], gr.n_relations, P, seed=1, epoch=e_now)
    assert owners == o_now.tolist()


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("model", ["transe_l2", "distmult"])
def test_dist_head_owner_placement_locality(model, P):
    # reading c.13'': the graph renumbered by kge_locality_order, head-owner placement and local
    # negatives: every head row and every uniform negative is local; parity with the oracle's P-rank union step
    gr = synth.graph("tiny")
    h0, r0, t0 = gr.triples()
    nid, cut = kge.locality_order(h0, t0, gr.n_entities, P)
    trip = (nid[h0], r0, nid[t0])
    B, g, k, d = 128, 32, 32, 32
    cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=d, batch_size=B,
                     chunk_size=g, neg_k=k, placement=1, neg_local=1, neg_precision="fp32")
    hs = kge.init_local_group(cfg, P, *trip)
    orc = O.Trainer(model, gr.n_entities, gr.n_relations, d, B, g, k, world_size=P, triples=trip, placement=1,
                    neg_local=1)
    for w in range(P):
        s = hs[w].sample(2)
        assert np.array_equal(s["pos"], orc.sample(2, w)[0]) and np.all(trip[0][s["pos"]] % P == w)
        assert np.all(s["neg"] % P == w)
    steps = 20
    for _ in range(steps):
        for h in hs:
            h.train_step(1, return_loss=False)
    lg = sum(h.read_losses(0, steps).astype(np.float64) for h in hs)
    lo = orc.train(steps)
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= 1e-5
    ids, rids = np.arange(gr.n_entities), np.arange(gr.n_relations)
    got = np.stack([hs[e % P].get_rows(0, [e])[0] for e in ids])
    assert np.abs(got - orc.get_rows(0, ids)).max() <= 1e-4
    rel = hs[0].get_rows(1, rids)  # every relation replicated: all replicas agree with the union step
    assert np.abs(rel - orc.get_rows(1, rids)).max() <= 1e-4
    assert all(np.array_equal(rel, h.get_rows(1, rids)) for h in hs[1:])
