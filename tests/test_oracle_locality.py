"""Pins of reading c.13'' (PAPER.md:395-406 [3.2] METIS partitioning, "assign a METIS partition
(all entities and triplets incident to the entities) to a machine"): the built-in BFS-grown balanced partitioner
(SPEC's partition_graph_greedy substitute for METIS) with the renumbering that puts part w on rank w's shard, and
head-owner triple placement. Examples from SPEC (two bridged 4-cliques, P = 1, clustered graph vs random parts)."""
import numpy as np
import pytest

import oracle as O


def _cliques_bridge():
    e = [(a, b) for a in range(4) for b in range(a + 1, 4)] + [(a, b) for a in range(4, 8) for b in range(a + 1, 8)]
    e.append((3, 4))
    return np.array([x[0] for x in e]), np.array([x[1] for x in e])


def test_two_cliques_bridge_cut_one():
    # SPEC: two 4-cliques joined by one bridge edge, P = 2 -> edge cut 1 (the balanced optimum)
    h, t = _cliques_bridge()
    nid, part, cut = O.locality_order(h, t, 8, 2)
    assert cut == 1 and part.tolist() == [0, 0, 0, 0, 1, 1, 1, 1]
    # part w lands on rank w's shard (owner = new id mod P), ids a permutation
    assert sorted(nid.tolist()) == list(range(8)) and np.all(nid % 2 == part)


def test_single_part():
    h, t = _cliques_bridge()
    nid, part, cut = O.locality_order(h, t, 8, 1)
    assert cut == 0 and not part.any() and np.array_equal(nid, np.arange(8))


@pytest.mark.parametrize("P", [3, 10])
def test_clustered_graph_beats_random(P):
    # SPEC: 1000 entities in 10 dense clusters with sparse inter-cluster edges: the BFS parts cut far fewer triples
    # than random parts of the same sizes (~(1 - 1/P) of all edges)
    rng = np.random.default_rng(0)
    cl = np.repeat(np.arange(10), 100)
    h = rng.integers(0, 1000, 20000)
    same = rng.random(20000) < 0.97
    t = np.where(same, cl[h] * 100 + rng.integers(0, 100, 20000), rng.integers(0, 1000, 20000))
    nid, part, cut = O.locality_order(h, t, 1000, P)
    sizes = np.bincount(part, minlength=P)
    assert np.array_equal(sizes, [(1000 - w + P - 1) // P for w in range(P)])  # = the shard sizes
    assert sorted(nid.tolist()) == list(range(1000)) and np.all(nid % P == part)
    assert cut == int(np.sum(part[h] != part[t]))  # the reported cut is the counting loop
    rand_cuts = [np.sum(p[h] != p[t]) for p in (rng.permutation(part) for _ in range(20))]
    assert cut < 0.8 * min(rand_cuts), (cut, min(rand_cuts))  # SPEC: strictly below random (measured 0.51-0.71)


def test_head_owner_placement():
    # c.13'': with placement = 1 every rank's positives are the triples whose head it owns (h mod P)
    rng = np.random.default_rng(3)
    trip = rng.integers(0, 500, 3000), rng.integers(0, 7, 3000), rng.integers(0, 500, 3000)
    tr = O.Trainer("distmult", 500, 7, 8, 32, 8, 8, seed=2, world_size=4, triples=trip, placement=1)
    for w in range(4):
        for s in (0, 5, 93):
            pos, _, _ = tr.sample(s, w)
            assert np.all(trip[0][pos] % 4 == w)
    # an epoch visits each of the rank's triples once (Feistel permutation over its list)
    n0 = int(np.sum(trip[0] % 4 == 0))
    seen = np.concatenate([tr.sample(s, 0)[0] for s in range(n0 // 32)])
    assert len(np.unique(seen)) == len(seen)


@pytest.mark.parametrize("P", [2, 3, 8])
def test_library_locality_order_equals_oracle(P):
    # the library's host partitioner (kge_locality_order, independent code) gives the oracle's renumbering bit-exactly
    from paper_2004_08532_b200 import kge
    import synth
    gr = synth.graph("tiny")
    h, r, t = gr.triples()
    nid_o, part, cut_o = O.locality_order(h, t, gr.n_entities, P)
    nid_l, cut_l = kge.locality_order(h, t, gr.n_entities, P)
    assert np.array_equal(nid_o, nid_l) and cut_o == cut_l
