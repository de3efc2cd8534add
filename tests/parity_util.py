"""Helpers of the parity tests: per-pair oracle scores of a sampled step, the scale of reading c.14, the TransE-L1 kink
set of reading R-L1, and table synchronisation. Test infrastructure only (calls oracle/, never the CUDA path)."""
import os

import numpy as np

# the oracle's optional parallel loops give bit-identical results (oracle.cpp threads()); use the host's cores
os.environ.setdefault("ORC_THREADS", str(max(1, min(64, os.cpu_count() or 1))))

GAMMA = 12.0
TABLES = {"transr": ((0, 1, 2, 3, 4, 5)), "default": (0, 1, 3, 4)}


def tables_of(model):
    return TABLES["transr"] if model == "transr" else TABLES["default"]


def copy_tables(orc, gpu, model, n_e, n_r):
    """Teacher forcing: overwrite every GPU table with the oracle's (rounded to fp32)."""
    ids, rids = np.arange(n_e), np.arange(n_r)
    for tab in tables_of(model):
        gpu.set_rows(tab, ids if tab in (0, 3) else rids, orc.get_rows(tab, ids if tab in (0, 3) else rids))


def step_triples(orc, step, g):
    """The B x k negative triples of a step in the layout of kge_debug_neg_scores: row i = positive i, column j =
    negative slot j of its chunk; tail corruption (h_i, r_i, x_j), head corruption (x_j, r_i, t_i)."""
    pos, neg, mode = orc.sample(step)
    B = len(pos)
    k = len(neg) // len(mode)
    return pos, neg.reshape(len(mode), k), mode, B, k


def pair_scores(orc, step, heads, rels, tails, g):
    """Oracle f-_{i,j} of every negative pair of `step` (naive per-triple Table-1 score, c.8) and the c.14 scale S."""
    pos, neg, mode, B, k = step_triples(orc, step, g)
    h, r, t = heads[pos], rels[pos], tails[pos]
    C = len(mode)
    hh = np.empty((B, k), np.int64)
    tt = np.empty((B, k), np.int64)
    for c in range(C):
        sl = slice(c * g, (c + 1) * g)
        if mode[c] == 0:  # tail corruption
            hh[sl] = h[sl, None]
            tt[sl] = neg[c][None, :]
        else:
            hh[sl] = neg[c][None, :]
            tt[sl] = t[sl, None]
    rr = np.repeat(r[:, None], k, 1)
    f = orc.score_triples(hh.ravel(), rr.ravel(), tt.ravel()).reshape(B, k)
    return f, (pos, neg, mode, h, r, t)


def dot_scale(model, orc, meta, g):
    """S = sum of |terms| of the dot score for every pair (reading c.14), computed chunk by chunk as a product of
    absolute values."""
    pos, neg, mode, h, r, t = meta
    B, k = len(pos), neg.shape[1]
    S = np.empty((B, k))
    for c in range(len(mode)):
        sl = slice(c * g, (c + 1) * g)
        R = orc.get_rows(1, r[sl])
        X = np.abs(orc.get_rows(0, neg[c]))
        other = orc.get_rows(0, h[sl] if mode[c] == 0 else t[sl])  # the uncorrupted entity
        if model == "distmult":
            S[sl] = np.abs(other * R) @ X.T
        else:  # complex, rows [re | im]
            n = R.shape[1] // 2
            ar, ai, rr_, ri = other[:, :n], other[:, n:], R[:, :n], R[:, n:]
            # tail (x = t): t_r (|hr rr| + |hi ri|), t_i (|hi rr| + |hr ri|); head (x = h): h_r (|rr tr| + |ri ti|),
            # h_i (|rr ti| + |ri tr|) -- the same expression with (a_r, a_i) the uncorrupted entity
            A = np.concatenate([np.abs(ar * rr_) + np.abs(ai * ri), np.abs(ai * rr_) + np.abs(ar * ri)], 1)
            S[sl] = A @ X.T
    return S


def check_pair_scores(model, got, ref, meta, orc, g, rtol, gamma=GAMMA):
    """|f - f_ref| <= rtol * max(|f_ref|, S) element by element (reading c.14). Returns the worst ratio."""
    if model in ("distmult", "complex"):
        S = dot_scale(model, orc, meta, g)
    else:
        S = abs(gamma) + np.abs(gamma - ref)
    err = np.abs(got.astype(np.float64) - ref) / np.maximum(np.abs(ref), S)
    assert np.all(np.isfinite(got)), "captured scores contain non-finite values"
    return float(err.max())


def l1_kink_coords(orc, meta, g, n_e, n_r, d):
    """Reading R-L1: coordinates whose TransE-L1 subgradient sign may legitimately differ between the fp32 kernels and
    the fp64 oracle -- some pair difference (h + r - x, x - (t - r), or h + r - t) lies within fp32 rounding of 0
    (|diff| <= 2^-21 (|a| + |b| + |c|)). Returns boolean masks [n_e, d] and [n_r, d] of the rows' coordinates whose
    gradient such a pair touches."""
    pos, neg, mode, h, r, t = meta
    ke = np.zeros((n_e, d), bool)
    kr = np.zeros((n_r, d), bool)
    H, R, T = orc.get_rows(0, h), orc.get_rows(1, r), orc.get_rows(0, t)
    tau = 2.0 ** -21
    pk = np.abs(H + R - T) <= tau * (np.abs(H) + np.abs(R) + np.abs(T))
    for a, ids in ((ke, h), (kr, r), (ke, t)):
        np.logical_or.at(a, ids, pk)
    for c in range(len(mode)):
        sl = slice(c * g, (c + 1) * g)
        X = orc.get_rows(0, neg[c])
        if mode[c] == 0:
            O, mag = H[sl] + R[sl], np.abs(H[sl]) + np.abs(R[sl])
        else:
            O, mag = T[sl] - R[sl], np.abs(T[sl]) + np.abs(R[sl])
        for i0 in range(0, O.shape[0], 32):  # [32, k, d] blocks
            diff = np.abs(O[i0:i0 + 32, None, :] - X[None, :, :])
            kink = diff <= tau * (mag[i0:i0 + 32, None, :] + np.abs(X)[None, :, :])
            np.logical_or.at(ke, neg[c], kink.any(0))
            rows_i = kink.any(1)
            ii = np.arange(c * g + i0, c * g + min(i0 + 32, O.shape[0]))
            np.logical_or.at(kr, r[ii], rows_i)
            np.logical_or.at(ke, (h if mode[c] == 0 else t)[ii], rows_i)
    return ke, kr
