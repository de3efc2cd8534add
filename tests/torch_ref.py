"""Independent float64 torch re-derivation of Table 1 + logistic loss (c.9) +
Adagrad (c.11), used ONLY to pin the oracle (its hand-derived gradients, dedup-sum and wiring) through autograd."""
import torch


def score(model, h, r, t, M=None, variant=0, gamma=0.0):
    """Batched over leading dims; last dim = features."""
    d = h.shape[-1]
    n = d // 2
    if model == "transe_l1":
        return gamma - (h + r - t).abs().sum(-1)
    if model == "transe_l2":
        return gamma - torch.linalg.vector_norm(h + r - t, dim=-1)
    if model == "distmult":
        return (h * r * t).sum(-1)
    if model == "complex":
        hc = torch.complex(h[..., :n], h[..., n:])
        rc = torch.complex(r[..., :n], r[..., n:])
        tc = torch.complex(t[..., :n], t[..., n:])
        return (hc * rc * tc.conj()).sum(-1).real
    if model == "rotate":
        hc = torch.complex(h[..., :n], h[..., n:])
        tc = torch.complex(t[..., :n], t[..., n:])
        rc = torch.polar(torch.ones_like(r), r)
        z = hc * rc - tc
        m2 = z.real ** 2 + z.imag ** 2
        return gamma - (m2.sum(-1) if variant == 0 else m2.sqrt().sum(-1))
    if model == "transr":
        p = (M @ h.unsqueeze(-1)).squeeze(-1) + r - (M @ t.unsqueeze(-1)).squeeze(-1)
        return gamma - (p ** 2).sum(-1)
    if model == "rescal":  # h^T M_r t; no relation vector
        return (h * (M @ t.unsqueeze(-1)).squeeze(-1)).sum(-1) + 0.0 * r.sum(-1)
    raise ValueError(model)


def step_loss(model, E, R, Pj, samples, triples, B, g, k, gamma, variant, loss="logistic"):
    """samples: list over ranks of (pos_idx, neg, mode). Loss = sum over ranks of the c.9 logistic loss, or of the
    c.9' pairwise ranking loss sum_i sum_j relu(gamma - f+_i + f-_ij) / (B k)."""
    h_all, r_all, t_all = triples
    total = 0.0
    for pos, neg, mode in samples:
        hh = torch.as_tensor(h_all[pos])
        rr = torch.as_tensor(r_all[pos])
        tt = torch.as_tensor(t_all[pos])
        M = Pj[rr] if Pj is not None else None
        fpos = score(model, E[hh], R[rr], E[tt], M, variant, gamma)
        C = B // g
        negs = torch.as_tensor(neg).view(C, k)
        fneg = []
        for i in range(B):
            c = i // g
            x = negs[c]
            Mi = M[i].expand(k, -1, -1) if M is not None else None
            if mode[c] == 0:
                f = score(model, E[hh[i]].expand(k, -1), R[rr[i]].expand(k, -1), E[x], Mi, variant, gamma)
            else:
                f = score(model, E[x], R[rr[i]].expand(k, -1), E[tt[i]].expand(k, -1), Mi, variant, gamma)
            fneg.append(f)
        fneg = torch.stack(fneg)
        if loss == "pairwise":
            total = total + torch.relu(gamma - fpos[:, None] + fneg).sum() / (B * k)
            continue
        lp = torch.nn.functional.logsigmoid(fpos).sum()
        ln = torch.nn.functional.logsigmoid(-fneg).sum()
        total = total - lp / B - ln / (B * k)
    return total


def adagrad_(W, S, G, lr, eps):
    """Row-wise Adagrad on every row (rows with zero gradient are unchanged)."""
    w = W.shape[1] if W.dim() == 2 else W[0].numel()
    G2 = G.reshape(G.shape[0], -1)
    S += (G2 * G2).sum(1) / w
    W -= (lr * G2 / torch.sqrt(S + eps).unsqueeze(1)).reshape(W.shape)
