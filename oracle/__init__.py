"""ctypes binding of liboracle.so -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may import this.
The product package paper_2004_08532_b200 never imports it (tests/test_abi.py checks that).
See oracle.h for what each function follows in PAPER.md / SURVEY.md 8(c).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .build import LIB
from .build import build as build_lib

TRANSE_L1, TRANSE_L2, DISTMULT, COMPLEX, ROTATE, TRANSR, RESCAL = range(7)
MODEL_IDS = {"transe_l1": 0, "transe_l2": 1, "distmult": 2, "complex": 3, "rotate": 4, "transr": 5, "rescal": 6}
TAIL, HEAD, ALTERNATE = 0, 1, 2

P = ctypes.POINTER
_i64p = P(ctypes.c_int64)
_dp = P(ctypes.c_double)


class Config(ctypes.Structure):
    _fields_ = [("model", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("n_entities", ctypes.c_int64), ("n_relations", ctypes.c_int64),
                ("dim", ctypes.c_int32), ("batch", ctypes.c_int32), ("chunk", ctypes.c_int32),
                ("neg_k", ctypes.c_int32),
                ("gamma", ctypes.c_float), ("lr", ctypes.c_float), ("eps", ctypes.c_float),
                ("init_bound", ctypes.c_float), ("seed", ctypes.c_uint64), ("corrupt", ctypes.c_int32),
                ("rotate_variant", ctypes.c_int32), ("world_size", ctypes.c_int32), ("lazy_rows", ctypes.c_int32),
                ("lag", ctypes.c_int32), ("neg_deg_k", ctypes.c_int32), ("neg_local", ctypes.c_int32),
                ("loss", ctypes.c_int32), ("repartition", ctypes.c_int32), ("placement", ctypes.c_int32)]


TRIPLE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int64, _i64p, _i64p, _i64p)

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build_lib()
        L = ctypes.CDLL(LIB)
        L.orc_philox.argtypes = [P(ctypes.c_uint32), P(ctypes.c_uint32), P(ctypes.c_uint32)]
        L.orc_feistel_index.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64]
        L.orc_feistel_index.restype = ctypes.c_uint64
        L.orc_neg_id.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]
        L.orc_neg_id.restype = ctypes.c_int64
        L.orc_mode.argtypes = [ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint32]
        L.orc_mode.restype = ctypes.c_int32
        L.orc_init_value.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_float]
        L.orc_init_value.restype = ctypes.c_float
        L.orc_default_bound.argtypes = [ctypes.c_float, ctypes.c_int32]
        L.orc_default_bound.restype = ctypes.c_float
        L.orc_relation_partition.argtypes = [_i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, P(ctypes.c_int32)]
        L.orc_relation_partition.restype = ctypes.c_int32
        L.orc_relation_partition_epoch.argtypes = [_i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                                   ctypes.c_uint64, ctypes.c_uint32, P(ctypes.c_int32)]
        L.orc_relation_partition_epoch.restype = ctypes.c_int32
        L.orc_locality_order.argtypes = [_i64p, _i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, _i64p,
                                         P(ctypes.c_int32)]
        L.orc_locality_order.restype = ctypes.c_int64
        L.orc_rank_triples.argtypes = [_i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _i64p]
        L.orc_rank_triples.restype = ctypes.c_int64
        L.orc_score.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_int32, _dp, _dp, _dp, _dp]
        L.orc_score.restype = ctypes.c_double
        _fp = P(ctypes.c_float)
        L.orc_score_f.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_float, ctypes.c_int32, _fp, _fp, _fp, _fp]
        L.orc_score_f.restype = ctypes.c_float
        L.orc_score_grad.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_int32, _dp, _dp, _dp,
                                     _dp, ctypes.c_double, _dp, _dp, _dp, _dp]
        L.orc_score_group.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_int32, ctypes.c_int32, _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc_logistic_loss.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                        _dp, _dp]
        L.orc_logistic_loss.restype = ctypes.c_double
        L.orc_ranking_loss.argtypes = [_dp, _dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, _dp, _dp]
        L.orc_ranking_loss.restype = ctypes.c_double
        L.orc_eval_candidates.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, _i64p, _i64p, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, _i64p, P(ctypes.c_int32)]
        L.orc_adagrad.argtypes = [_dp, _dp, _dp, ctypes.c_int32, ctypes.c_double, ctypes.c_double]
        L.orc_dedup.argtypes = [_i64p, ctypes.c_int64, _i64p, P(ctypes.c_int32), _i64p, _i64p]
        L.orc_dedup.restype = ctypes.c_int64
        L.orc_create.argtypes = [P(Config), _i64p, _i64p, _i64p, ctypes.c_int64, TRIPLE_FN, ctypes.c_void_p]
        L.orc_create.restype = ctypes.c_void_p
        L.orc_destroy.argtypes = [ctypes.c_void_p]
        L.orc_sample.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, _i64p, _i64p, P(ctypes.c_int8)]
        L.orc_occurrences.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, _i64p, _i64p]
        L.orc_train.argtypes = [ctypes.c_void_p, ctypes.c_int64, _dp]
        L.orc_flush.argtypes = [ctypes.c_void_p]
        L.orc_get_rows.argtypes = [ctypes.c_void_p, ctypes.c_int32, _i64p, ctypes.c_int64, _dp]
        L.orc_set_rows.argtypes = [ctypes.c_void_p, ctypes.c_int32, _i64p, ctypes.c_int64, _dp]
        L.orc_score_triples.argtypes = [ctypes.c_void_p, _i64p, _i64p, _i64p, ctypes.c_int64, _dp]
        L.orc_next_step.argtypes = [ctypes.c_void_p]
        L.orc_next_step.restype = ctypes.c_int64
        L.orc_set_step.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        L.orc_table_width.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        L.orc_table_width.restype = ctypes.c_int32
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(P(ct)) if a is not None else None


def d64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().orc_philox(c, k, o)
    return list(o)


def feistel_index(n, seed, epoch, p):
    return lib().orc_feistel_index(n, seed, epoch, p)


def neg_id(seed, n_ent, step, cg, j):
    return lib().orc_neg_id(seed, n_ent, step, cg, j)


def mode(corrupt, step, cg):
    return lib().orc_mode(corrupt, step, cg)


def init_value(seed, table, row, col, bound):
    return lib().orc_init_value(seed, table, row, col, bound)


def default_bound(gamma, dim):
    return lib().orc_default_bound(gamma, dim)


def rel_width(model, d):
    return d // 2 if model == ROTATE else d


def score(model, h, r, t, M=None, gamma=0.0, variant=0):
    h, r, t = d64(h), d64(r), d64(t)
    Mp = d64(M) if M is not None else None
    return lib().orc_score(model, variant, gamma, len(h), _p(h, ctypes.c_double), _p(r, ctypes.c_double),
                           _p(t, ctypes.c_double), _p(Mp, ctypes.c_double))


def score_f(model, h, r, t, M=None, gamma=0.0, variant=0):
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    h, r, t = f32(h), f32(r), f32(t)
    Mp = f32(M) if M is not None else None
    return lib().orc_score_f(model, variant, gamma, len(h), _p(h, ctypes.c_float), _p(r, ctypes.c_float),
                             _p(t, ctypes.c_float), _p(Mp, ctypes.c_float))


def score_grad(model, h, r, t, M=None, upstream=1.0, gamma=0.0, variant=0):
    h, r, t = d64(h), d64(r), d64(t)
    Mp = d64(M) if M is not None else None
    dh, dr, dt = np.zeros_like(h), np.zeros_like(r), np.zeros_like(t)
    dM = np.zeros_like(Mp) if Mp is not None else None
    dp = lambda a: _p(a, ctypes.c_double)
    lib().orc_score_grad(model, variant, gamma, len(h), dp(h), dp(r), dp(t), dp(Mp), upstream, dp(dh), dp(dr),
                         dp(dt), dp(dM))
    return dh, dr, dt, dM


def score_group(model, mode_, H, R, T, X, M=None, gamma=0.0, variant=0):
    H, R, T, X = d64(H), d64(R), d64(T), d64(X)
    g, d = H.shape
    k = X.shape[0]
    Mp = d64(M) if M is not None else None
    out = np.zeros((g, k))
    dp = lambda a: _p(a, ctypes.c_double)
    lib().orc_score_group(model, variant, gamma, d, mode_, g, k, dp(H), dp(R), dp(T), dp(Mp), dp(X), dp(out))
    return out


def logistic_loss(pos, neg, B, k):
    pos, neg = d64(pos), d64(neg)
    dpos, dneg = np.zeros_like(pos), np.zeros_like(neg)
    dp = lambda a: _p(a, ctypes.c_double)
    L = lib().orc_logistic_loss(dp(pos), len(pos), dp(neg), len(neg), B, k, dp(dpos), dp(dneg))
    return L, dpos, dneg


def ranking_loss(pos, neg, k, gamma):
    """c.9' pairwise ranking loss: pos[B], neg[B*k] (row i = positive i's negatives)."""
    pos, neg = d64(pos), d64(neg)
    B = len(pos)
    dpos, dneg = np.zeros_like(pos), np.zeros_like(neg)
    dp = lambda a: _p(a, ctypes.c_double)
    L = lib().orc_ranking_loss(dp(pos), dp(neg), B, k, float(gamma), dp(dpos), dp(dneg))
    return L, dpos, dneg


LOSSES = {"logistic": 0, "pairwise": 1}


def adagrad(row, state, g, lr, eps=1e-10):
    row, g = d64(row).copy(), d64(g)
    st = np.array([state], dtype=np.float64)
    dp = lambda a: _p(a, ctypes.c_double)
    lib().orc_adagrad(dp(row), dp(st), dp(g), len(row), lr, eps)
    return row, float(st[0])


def dedup(ids):
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    n = len(ids)
    uniq = np.zeros(n, np.int64)
    inv = np.zeros(n, np.int32)
    seg_off = np.zeros(n + 1, np.int64)
    seg_occ = np.zeros(n, np.int64)
    nu = lib().orc_dedup(_p(ids, ctypes.c_int64), n, _p(uniq, ctypes.c_int64), _p(inv, ctypes.c_int32),
                         _p(seg_off, ctypes.c_int64), _p(seg_occ, ctypes.c_int64))
    return uniq[:nu], inv, seg_off[:nu + 1], seg_occ


def relation_partition(rels, n_rel, P_, seed=None, epoch=None):
    """c.13 relation partition; with seed and epoch: the randomised partition of that epoch (c.13')."""
    rels = np.ascontiguousarray(rels, dtype=np.int64)
    owner = np.zeros(n_rel, np.int32)
    if epoch is None:
        ns = lib().orc_relation_partition(_p(rels, ctypes.c_int64), len(rels), n_rel, P_, _p(owner, ctypes.c_int32))
    else:
        ns = lib().orc_relation_partition_epoch(_p(rels, ctypes.c_int64), len(rels), n_rel, P_, int(seed), int(epoch),
                                                _p(owner, ctypes.c_int32))
    return owner, ns


def locality_order(heads, tails, n_entities, P_):
    """c.13'' BFS-grown balanced parts (SPEC partition_graph_greedy) and the shard renumbering: (new_id, part, cut)."""
    h, t = np.ascontiguousarray(heads, np.int64), np.ascontiguousarray(tails, np.int64)
    nid = np.zeros(n_entities, np.int64)
    part = np.zeros(n_entities, np.int32)
    cut = lib().orc_locality_order(_p(h, ctypes.c_int64), _p(t, ctypes.c_int64), len(h), n_entities, P_,
                                   _p(nid, ctypes.c_int64), _p(part, ctypes.c_int32))
    return nid, part, cut


def rank_triples(rels, n_rel, P_, rank):
    rels = np.ascontiguousarray(rels, dtype=np.int64)
    n = lib().orc_rank_triples(_p(rels, ctypes.c_int64), len(rels), n_rel, P_, rank, None)
    out = np.zeros(n, np.int64)
    lib().orc_rank_triples(_p(rels, ctypes.c_int64), len(rels), n_rel, P_, rank, _p(out, ctypes.c_int64))
    return out


class Trainer:
    """The oracle training step (lag 0), P ranks simulated as one union step (SURVEY c.12, c.13)."""

    def __init__(self, model, n_entities, n_relations, dim, batch, chunk, neg_k, gamma=12.0, lr=0.1, eps=1e-10,
                 init_bound=0.0, seed=1, corrupt=ALTERNATE, rotate_variant=0, world_size=1, precision=0,
                 triples=None, graph=None, lazy_rows=False, lag=0, neg_deg_k=0, neg_local=0, loss="logistic",
                 repartition=0, placement=0):
        if isinstance(model, str):
            model = MODEL_IDS[model]
        self.model = model
        self.cfg = Config(model, precision, n_entities, n_relations, dim, batch, chunk, neg_k, gamma, lr, eps,
                          init_bound, seed, corrupt, rotate_variant, world_size, int(lazy_rows), int(lag),
                          int(neg_deg_k), int(neg_local), LOSSES[loss] if isinstance(loss, str) else int(loss),
                          int(repartition), int(placement))
        self._keep = []
        if triples is not None:
            h, r, t = [np.ascontiguousarray(a, dtype=np.int64) for a in triples]
            self._keep = [h, r, t]
            self.h = lib().orc_create(ctypes.byref(self.cfg), _p(h, ctypes.c_int64), _p(r, ctypes.c_int64),
                                      _p(t, ctypes.c_int64), len(h), TRIPLE_FN(), None)
        else:
            import synth  # the shared input generator, through a callback
            gc = graph._c()
            L = synth.lib()

            def fn(ctx, i, hp, rp, tp):
                L.synth_triple(ctypes.byref(gc), i, hp, rp, tp)

            cb = TRIPLE_FN(fn)
            self._keep = [gc, cb]
            self.h = lib().orc_create(ctypes.byref(self.cfg), None, None, None, graph.n_triples, cb, None)
        if not self.h:
            raise ValueError("orc_create rejected the configuration")
        self.B, self.k, self.C = batch, neg_k, batch // chunk
        self.dim = dim

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def sample(self, step, rank=0):
        pos = np.zeros(self.B, np.int64)
        neg = np.zeros(self.C * self.k, np.int64)
        mode_ = np.zeros(self.C, np.int8)
        lib().orc_sample(self.h, step, rank, _p(pos, ctypes.c_int64), _p(neg, ctypes.c_int64),
                         _p(mode_, ctypes.c_int8))
        return pos, neg, mode_

    def occurrences(self, step, rank=0):
        e = np.zeros(2 * self.B + self.C * self.k, np.int64)
        r = np.zeros(self.B, np.int64)
        lib().orc_occurrences(self.h, step, rank, _p(e, ctypes.c_int64), _p(r, ctypes.c_int64))
        return e, r

    def train(self, n_steps):
        losses = np.zeros(n_steps)
        lib().orc_train(self.h, n_steps, _p(losses, ctypes.c_double))
        return losses

    def flush(self):
        """lag = 1: apply the held-back entity update of the last step."""
        lib().orc_flush(self.h)

    def width(self, table):
        return lib().orc_table_width(self.h, table)

    def get_rows(self, table, ids):
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        w = self.width(table)
        out = np.zeros((len(ids), w))
        rc = lib().orc_get_rows(self.h, table, _p(ids, ctypes.c_int64), len(ids), _p(out, ctypes.c_double))
        if rc != 0:
            raise ValueError(f"orc_get_rows rc={rc}")
        return out

    def set_rows(self, table, ids, rows):
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        rows = d64(rows)
        rc = lib().orc_set_rows(self.h, table, _p(ids, ctypes.c_int64), len(ids), _p(rows, ctypes.c_double))
        if rc != 0:
            raise ValueError(f"orc_set_rows rc={rc}")

    def score_triples(self, hs, rs, ts):
        hs, rs, ts = [np.ascontiguousarray(a, dtype=np.int64) for a in (hs, rs, ts)]
        out = np.zeros(len(hs))
        lib().orc_score_triples(self.h, _p(hs, ctypes.c_int64), _p(rs, ctypes.c_int64), _p(ts, ctypes.c_int64),
                                len(hs), _p(out, ctypes.c_double))
        return out

    @property
    def step(self):
        return lib().orc_next_step(self.h)

    def set_step(self, s):
        """Continue from step s (sampling is a pure function of (seed, step))."""
        lib().orc_set_step(self.h, int(s))


def eval_candidates(seed, n_entities, heads, tails, n_queries, n_uniform, n_degree, both):
    """Reading c.15' second-protocol candidates: per query n_uniform uniform and n_degree
    degree-proportional corruptions from the counter-based stream EVAL; returns (entities, sides) [n_queries x m]."""
    th, tt = np.ascontiguousarray(heads, np.int64), np.ascontiguousarray(tails, np.int64)
    m = n_uniform + n_degree
    ent = np.zeros((n_queries, m), np.int64)
    side = np.zeros((n_queries, m), np.int32)
    lib().orc_eval_candidates(int(seed), int(n_entities), len(th), _p(th, ctypes.c_int64), _p(tt, ctypes.c_int64),
                              n_queries, n_uniform, n_degree, int(both), _p(ent, ctypes.c_int64),
                              _p(side, ctypes.c_int32))
    return ent, side


def link_rank(trainer, hs, rs, ts, head=False, candidates=None, known=None):
    """Link-prediction ranks, PAPER.md:652-665 [5.3] step by step: for each positive triple build S_i = the positive
    plus its negative triples (every corruption of the tail -- head=True: the head; head="both": every corruption of
    the head AND of the tail in one list, as the paper's "(h', r, t) and (h, r, t')" -- or, second protocol, the given
    candidates; with `known` (a set of (h, r, t) tuples), first protocol filtered: corruptions that already exist in
    the dataset are removed), score S_i with Table 1, order it by non-increasing score with the positive LAST among
    equal scores (reading c.15), rank_i = the positive's 1-based position. candidates: per query an array of entity
    ids (one side), or with head="both" a pair (entities, sides: 0 = tail replaced, 1 = head replaced). The corruption
    equal to the positive itself is not a negative triple."""
    out = []
    n_e = trainer.cfg.n_entities
    both = isinstance(head, str) and head == "both"
    for i in range(len(hs)):
        h, r, t = int(hs[i]), int(rs[i]), int(ts[i])
        if both:
            if candidates is None:
                cs = [(e, 0) for e in range(n_e)] + [(e, 1) for e in range(n_e)]
            else:
                cs = [(int(e), int(sd)) for e, sd in zip(*candidates[i])]
            neg = [(e, r, t) if sd else (h, r, e) for e, sd in cs if e != (h if sd else t)]
        else:
            true_e = h if head else t
            ents = range(n_e) if candidates is None else [int(e) for e in candidates[i]]
            neg = [(e, r, t) if head else (h, r, e) for e in ents if e != true_e]
        if known is not None:
            neg = [x for x in neg if x not in known]
        trip = [(h, r, t)] + neg
        sc = trainer.score_triples([x[0] for x in trip], [x[1] for x in trip], [x[2] for x in trip])
        # non-increasing score; among equals the positive (index 0) goes last
        order = sorted(range(len(trip)), key=lambda j: (-sc[j], j == 0))
        out.append(order.index(0) + 1)
    return np.array(out, np.int64)


def link_metrics(ranks):
    """Hit@k, MR and MRR, PAPER.md:660-664 [5.3] formulas."""
    Q = len(ranks)
    if Q == 0:
        raise ValueError("metrics of an empty rank list")
    return {"Hit@1": sum(1 for x in ranks if x <= 1) / Q, "Hit@3": sum(1 for x in ranks if x <= 3) / Q,
            "Hit@10": sum(1 for x in ranks if x <= 10) / Q, "MR": sum(int(x) for x in ranks) / Q,
            "MRR": sum(1.0 / int(x) for x in ranks) / Q}
