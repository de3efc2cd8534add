"""SURVEY 8(f) item 4 variants on the CUDA path vs the CPU oracle (same seeded inputs, bars of reading c.14):
  - pairwise ranking loss (reading c.9'): every model, FFMA and tcgen05 paths, P = 2;
  - Table-1 RotatE on tcgen05 (the L2 expansion, PAPER.md:232 + 429-435) -- see also test_gpu_parity TC_MODELS.
"""
import numpy as np
import pytest

import oracle as O
import synth
from paper_2004_08532_b200 import kge
from tests import parity_util as U

pytestmark = pytest.mark.gpu


def _pair(model, d, B, g, k, precision="fp32", variant=0, graph="tiny", gamma=12.0, lr=0.1, loss="pairwise",
          world=1, init_bound=0.0):
    gr = synth.graph(graph)
    trip = gr.triples()
    cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=d, batch_size=B,
                     chunk_size=g, neg_k=k, gamma=gamma, lr=lr, seed=1, rotate_variant=variant,
                     neg_precision=precision, loss=loss, world_size=world, init_bound=init_bound)
    gpu = kge.init(cfg, *trip) if world == 1 else kge.init_local_group(cfg, world, *trip)
    orc = O.Trainer(model, gr.n_entities, gr.n_relations, d, B, g, k, gamma=gamma, lr=lr, seed=1,
                    rotate_variant=variant, triples=trip, loss=loss, world_size=world, init_bound=init_bound)
    return gr, trip, gpu, orc


# (model, variant, ranking margin gamma): with init_bound = 0.1 the step-0 score gaps f- - f+ of the tiny graph have a
# median ~0 and a 90th percentile of 0.69 / 0.093 / 0.003 / 0.0039 / 0.10 / 0.47 / 0.026 (L1, L2, DistMult, ComplEx,
# RotatE, RotatE modulus, TransR; oracle, measured once): gamma = half of it leaves ~60-70 % of the hinges active
PAIRWISE = [("transe_l1", 0, 0.35), ("transe_l2", 0, 0.05), ("distmult", 0, 0.0015), ("complex", 0, 0.002),
            ("rotate", 0, 0.05), ("rotate", 1, 0.25), ("transr", 0, 0.0125)]


def _hinges(orc, step, heads, rels, tails, g, gamma):
    """Oracle pair scores of `step` with the hinge margins m_ij = gamma - f+_i + f-_ij and their scale
    |gamma| + |f+_i| + |f-_ij| (reading c.14c)."""
    ref, meta = U.pair_scores(orc, step, heads, rels, tails, g)
    fpos = orc.score_triples(heads[meta[0]], rels[meta[0]], tails[meta[0]])
    m = gamma - fpos[:, None] + ref
    return ref, meta, m, abs(gamma) + np.abs(fpos)[:, None] + np.abs(ref)


def _loss_ok(lg, lo, m, scale, rtol):
    """Loss bar of reading c.14c: |L - L_ref| <= rtol * max(L_ref, S_L), S_L = mean over the active pairs of the
    hinge's scale (the loss is a mean of margins that shrink towards 0 while the scores they difference do not)."""
    act = m > 0
    S = (scale * act).sum() / m.size
    return abs(lg - lo) <= rtol * max(abs(lo), S), (lg, lo, S)


@pytest.mark.parametrize("model,variant,gamma", PAIRWISE)
@pytest.mark.parametrize("precision", ["fp32", "tf32"])
def test_pairwise_loss_parity(model, variant, gamma, precision):
    d = 32 if model == "transr" else 64
    lr = 0.05 if model == "transr" else 0.1
    gr, trip, gpu, orc = _pair(model, d, 256, 64, 64, precision=precision, variant=variant, gamma=gamma, lr=lr,
                               init_bound=0.1)
    heads, rels, tails = (np.asarray(a) for a in trip)
    tc = gpu.neg_path == "tf32"
    rtol = 2e-3 if tc else 1e-5
    ref, meta, m, scale = _hinges(orc, 0, heads, rels, tails, 64, gamma)
    # both sides of the hinge are exercised
    assert 0.05 < (m > 0).mean() < 0.999, (m > 0).mean()
    # step 0 on identical tables: per-pair scores element by element, then the loss
    gpu.set_option("capture_neg", 1)
    lg0 = gpu.train_step(1)[0]
    assert U.check_pair_scores(model, gpu.neg_scores(), ref, meta, orc, 64, rtol, gamma=gamma) <= rtol
    gpu.set_option("capture_neg", 0)
    lo0 = orc.train(1)[0]
    ok, info = _loss_ok(lg0, lo0, m, scale, rtol)
    assert ok, info
    # free-running: a hinge within rounding of 0 may be active on one side only, and Adagrad turns the flipped
    # gradient of a row into an O(lr) step (reading c.9' / R-L1), so the trajectories separate; the run must still
    # train as the oracle does. The strict per-step bars are teacher-forced (next test).
    lg, lo = gpu.train_step(39), orc.train(39)
    assert np.all(np.isfinite(lg))
    assert abs(np.log(lg[-1] / lo[-1])) <= 0.1, (lg[-1], lo[-1])


@pytest.mark.parametrize("precision", ["fp32", "tf32"])
@pytest.mark.parametrize("model", ["distmult", "transe_l2", "rotate", "transe_l1"])
def test_pairwise_teacher_forced_production_shape(model, precision):
    # configs[1]/[2] shapes (d = 400, B = 1024, g = k = 256): every step starts from the oracle's tables
    graph = "fb15k" if model in ("distmult", "transe_l2") else "wn18"
    gamma = {"distmult": 0.0015, "transe_l2": 0.05, "rotate": 0.05, "transe_l1": 0.35}[model]
    gr, trip, gpu, orc = _pair(model, 400, 1024, 256, 256, graph=graph, gamma=gamma, init_bound=0.1,
                               precision=precision)
    tc = gpu.neg_path == "tf32"
    assert tc == (precision == "tf32" and model != "transe_l1")
    heads, rels, tails = (np.asarray(a) for a in trip)
    ids, rids = np.arange(gr.n_entities), np.arange(gr.n_relations)
    worst_r, exempt = 0.0, 0
    for s in range(3):
        U.copy_tables(orc, gpu, model, gr.n_entities, gr.n_relations)
        ref, meta, m, scale = _hinges(orc, s, heads, rels, tails, 256, gamma)
        if model == "transe_l1" and not tc:  # kink coordinates of the tables this step starts from (reading R-L1)
            ke, kr = U.l1_kink_coords(orc, meta, 256, gr.n_entities, gr.n_relations, 400)
        lg, lo = gpu.train_step(1)[0], orc.train(1)[0]
        ok, info = _loss_ok(lg, lo, m, scale, 2e-3 if tc else 1e-5)
        assert ok, (s, info)
        dE = np.abs(gpu.get_rows(0, ids) - orc.get_rows(0, ids))
        dR = np.abs(gpu.get_rows(1, rids) - orc.get_rows(1, rids))
        if not tc:
            # the rows of pairs whose margin is within fp32 rounding of the hinge (and TransE-L1's kink coordinates)
            # may legitimately step differently; every other row meets 1e-4
            pos, neg, mode, h, r, t = meta
            near = np.abs(m) <= 2.0 ** -20 * scale
            ii, jj = np.nonzero(near)
            rows_e = set(h[ii]) | set(t[ii]) | set(neg.reshape(len(mode), -1)[ii // 256, jj])
            rows_r = set(r[ii])
            exempt += len(ii)
            if model == "transe_l1":
                dE, dR = np.where(ke, 0.0, dE), np.where(kr, 0.0, dR)
            dE[list(rows_e)] = 0.0
            dR[list(rows_r)] = 0.0
        worst_r = max(worst_r, dE.max(), dR.max())
    # FP32: 1e-4 (reading c.14); TF32: rows reported and loosely bounded (a hinge flipped by the TF32 score error moves
    # its rows by an Adagrad-normalised step)
    assert worst_r <= (5e-2 if tc else 1e-4), (model, worst_r, exempt)
    print(f"pairwise {model} {precision}: worst row {worst_r:.2e}, near-hinge pairs exempted {exempt}")


@pytest.mark.parametrize("model", ["distmult", "transe_l2"])
def test_pairwise_multi_rank(model):
    # P = 2 (single-device emulation): union-batch semantics of reading c.13 under the ranking loss
    gamma = 0.0015 if model == "distmult" else 0.05
    gr, trip, hs, orc = _pair(model, 32, 128, 32, 32, gamma=gamma, world=2, init_bound=0.1)
    lo = orc.train(10)
    lg = np.zeros(10)
    for _ in range(10):
        for h in hs:
            h.train_step(1, return_loss=False)
    for w, h in enumerate(hs):
        lg += h.read_losses(0, 10)
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= 1e-5, (lg, lo)


# ---------------------------------------------------------------- RESCAL (Table 1: h^T M_r t)
@pytest.mark.parametrize("precision", ["fp32", "tf32"])
@pytest.mark.parametrize("loss", ["logistic", "pairwise"])
def test_rescal_parity(precision, loss):
    # o = M_r^T h (tail) / M_r t (head), then the dot family's chunked negatives (FFMA or tcgen05); dM per unique
    # relation in a fixed order, one Adagrad state per matrix
    gamma = 12.0 if loss == "logistic" else 0.002
    gr, trip, gpu, orc = _pair("rescal", 32, 256, 64, 64, precision=precision, gamma=gamma, loss=loss,
                               init_bound=0.1 if loss == "pairwise" else 0.0, lr=0.05)
    assert gpu.neg_path == precision.replace("fp32", "ffma")
    heads, rels, tails = (np.asarray(a) for a in trip)
    rng = np.random.default_rng(1)
    q = rng.integers(0, gr.n_triples, 300)
    tol = 1e-5 if precision == "fp32" else 2e-3
    f, ref = gpu.score(heads[q], rels[q], tails[q]), orc.score_triples(heads[q], rels[q], tails[q])
    assert np.max(np.abs(f - ref)) <= 1e-5 * max(1.0, np.abs(ref).max())
    # per-pair negative scores of step 0
    gpu.set_option("capture_neg", 1)
    ref0, meta = U.pair_scores(orc, 0, heads, rels, tails, 64)
    lg = gpu.train_step(1)
    got = gpu.neg_scores()
    S = np.abs(ref0).max() + 1e-3
    assert np.max(np.abs(got - ref0)) <= tol * S, np.max(np.abs(got - ref0))
    gpu.set_option("capture_neg", 0)
    n = 30
    lg = np.concatenate([lg, gpu.train_step(n - 1)])
    lo = orc.train(n)
    rel = np.abs(lg - lo) / np.abs(lo)
    if loss == "logistic":
        assert rel.max() <= tol, (rel.max(), int(np.argmax(rel)))
    else:  # reading c.9': strict first steps, then the hinge flips separate the trajectories
        assert rel[:3].max() <= tol and abs(np.log(lg[-1] / lo[-1])) <= 0.1
    if loss == "logistic":
        ids, rids = np.arange(gr.n_entities), np.arange(gr.n_relations)
        rtol = 1e-4 if precision == "fp32" else 2e-2
        assert np.abs(gpu.get_rows(0, ids) - orc.get_rows(0, ids)).max() <= rtol
        assert np.abs(gpu.get_rows(2, rids) - orc.get_rows(2, rids)).max() <= rtol
        ps = orc.get_rows(5, rids)
        assert np.abs(gpu.get_rows(5, rids) - ps).max() <= (1e-6 if precision == "fp32" else 2e-3) * max(1.0, ps.max())
        # no relation vector: table 1 keeps its initial rows, its Adagrad states stay 0
        assert not gpu.get_rows(4, rids).any()


def test_rescal_teacher_forced_and_multi_rank():
    # FB15k-shaped graph at d = 64: one FP32 step from the oracle's tables at a time (rows 1e-4), then P = 2
    gr, trip, gpu, orc = _pair("rescal", 64, 1024, 256, 256, graph="fb15k", lr=0.05)
    ids, rids = np.arange(gr.n_entities), np.arange(gr.n_relations)
    for s in range(3):
        U.copy_tables(orc, gpu, "transr", gr.n_entities, gr.n_relations)  # every table incl. the projections
        lg, lo = gpu.train_step(1)[0], orc.train(1)[0]
        assert abs(lg - lo) / abs(lo) <= 1e-5
        assert np.abs(gpu.get_rows(0, ids) - orc.get_rows(0, ids)).max() <= 1e-4
        assert np.abs(gpu.get_rows(2, rids) - orc.get_rows(2, rids)).max() <= 1e-4
    gr, trip, hs, orc = _pair("rescal", 16, 128, 32, 32, world=2, lr=0.05)
    for _ in range(10):
        for h in hs:
            h.train_step(1, return_loss=False)
    lg = sum(h.read_losses(0, 10).astype(np.float64) for h in hs)
    lo = orc.train(10)
    assert np.max(np.abs(lg - lo) / np.abs(lo)) <= 1e-5
    ids = np.arange(gr.n_entities)
    got = np.stack([hs[e % 2].get_rows(0, [e])[0] for e in ids])
    assert np.abs(got - orc.get_rows(0, ids)).max() <= 1e-4
