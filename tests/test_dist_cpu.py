"""P > 1 host-side logic on CPU (no GPU): the library's relation partition (kge_partition, PAPER.md:476-495 [3.4],
reading c.13) against the oracle's independent implementation, and the world_size-2 exchange plumbing over gloo."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O
from paper_2004_08532_b200 import kge


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_partition_matches_oracle(P):
    rng = np.random.default_rng(P)
    n_rel = 300
    rels = np.minimum(rng.zipf(1.5, 30000) - 1, n_rel - 1)
    lists = []
    for w in range(P):
        owner, lst = kge.partition(rels, n_rel, P, w)
        o_owner, _ = O.relation_partition(rels, n_rel, P)
        assert np.array_equal(owner, o_owner)
        assert np.array_equal(lst, O.rank_triples(rels, n_rel, P, w))
        lists.append(lst)
    allidx = np.sort(np.concatenate(lists))
    assert np.array_equal(allidx, np.arange(len(rels)))  # every triple exactly once


def test_partition_spec_example_and_errors():
    rels = np.repeat(np.arange(4), [5, 4, 3, 2])
    owner, l0 = kge.partition(rels, 4, 2, 0)
    _, l1 = kge.partition(rels, 4, 2, 1)
    assert owner.tolist() == [0, 1, 1, 0] and (len(l0), len(l1)) == (7, 7)
    with pytest.raises(kge.KgeError):
        kge.partition(np.array([0, 7]), 4, 2, 0)  # relation id out of range


class _FakeHandle:
    """Stands in for a GPU handle: export() returns a rank-tagged blob, connect() records what it received."""

    def __init__(self, rank, world):
        self.cfg = kge.Config(world_size=world, rank=rank)
        self.rank = rank
        self.got = None

    def export(self):
        return bytes([self.rank]) * 128

    def connect(self, blobs):
        self.got = blobs


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    h = _FakeHandle(rank, world)
    kge.exchange_and_connect(h, dist.all_gather_object)
    rng = np.random.default_rng(0)
    rels = np.minimum(rng.zipf(1.4, 5000) - 1, 99)
    _, lst = kge.partition(rels, 100, world, rank)
    sizes = [None] * world
    dist.all_gather_object(sizes, lst.tolist())
    union = sorted(x for l in sizes for x in l)
    ok_blobs = [b[0] for b in h.got] == list(range(world)) and all(len(b) == 128 for b in h.got)
    q.put((rank, ok_blobs, union == list(range(len(rels)))))
    dist.destroy_process_group()


def test_gloo_world2_exchange_and_partition():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] and r[2] for r in res), res
