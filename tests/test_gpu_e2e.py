"""The pipelined caller-batch API (kge_train_batch_async): CUDA graphs per given slot, the sample of batch s+1 on its
own stream overlapping step s, and the step's loss stored by the device straight into a pinned host float (a
pageable target keeps the copy). Same results as the synchronous call, bit for bit."""
import numpy as np
import pytest
import torch

import synth
from paper_2004_08532_b200 import kge

pytestmark = pytest.mark.gpu


def _handle(model="transe_l2", precision="tf32"):
    gr = synth.graph("tiny")
    trip = gr.triples()
    cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=64, batch_size=256,
                     chunk_size=64, neg_k=64, gamma=12.0, lr=0.1, seed=1, neg_precision=precision)
    return gr, trip, kge.init(cfg, *trip)


@pytest.mark.parametrize("model,precision", [("transe_l2", "tf32"), ("distmult", "tf32"), ("rotate", "fp32")])
def test_async_pinned_loss_equals_sync(model, precision):
    gr, trip, ha = _handle(model, precision)
    _, _, hb = _handle(model, precision)
    n, B = 24, 256
    rng = np.random.default_rng(5)
    idx = rng.integers(0, gr.n_triples, size=(n, B))
    pinned = torch.empty((3, n, B), dtype=torch.int64, pin_memory=True)
    for a, arr in enumerate(trip):
        pinned[a].copy_(torch.from_numpy(np.ascontiguousarray(arr[idx])))
    loss = torch.full((n,), float("nan"), dtype=torch.float32, pin_memory=True)
    for st in range(n):
        o = st * B * 8
        ha.train_batch_async_ptr(pinned[0].data_ptr() + o, pinned[1].data_ptr() + o, pinned[2].data_ptr() + o,
                                 loss.data_ptr() + 4 * st)
    ha.sync()
    ref = np.array([hb.train_batch(trip[0][idx[st]], trip[1][idx[st]], trip[2][idx[st]]) for st in range(n)],
                   dtype=np.float32)
    assert np.array_equal(loss.numpy(), ref)
    ids = np.arange(gr.n_entities)
    assert np.array_equal(ha.get_rows(0, ids), hb.get_rows(0, ids))


def test_async_without_loss_pointer_still_trains():
    gr, trip, ha = _handle()
    _, _, hb = _handle()
    n, B = 10, 256
    pinned = torch.empty((3, n, B), dtype=torch.int64, pin_memory=True)
    idx = np.arange(n * B).reshape(n, B) % gr.n_triples
    for a, arr in enumerate(trip):
        pinned[a].copy_(torch.from_numpy(np.ascontiguousarray(arr[idx])))
    for st in range(n):
        o = st * B * 8
        ha.train_batch_async_ptr(pinned[0].data_ptr() + o, pinned[1].data_ptr() + o, pinned[2].data_ptr() + o, 0)
        hb.train_batch(trip[0][idx[st]], trip[1][idx[st]], trip[2][idx[st]])
    ha.sync()
    ids = np.arange(gr.n_entities)
    assert np.array_equal(ha.get_rows(0, ids), hb.get_rows(0, ids))
