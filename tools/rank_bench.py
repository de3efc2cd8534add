"""Throughput of link-prediction ranking (kge_rank, all-entity first protocol, raw and filtered) on an FB15k-shaped
table: queries/s and candidate scores/s. Run once per KGE_RANK_QB setting (the kernel choice is read once).

    python tools/rank_bench.py [model] [n_queries]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2004_08532_b200 import kge  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "transe_l2"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
gr = synth.graph("fb15k")
trip = gr.triples()
cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=400, batch_size=1024,
                 chunk_size=256, neg_k=256, gamma=12.0, lr=0.1, seed=1)
h = kge.init(cfg, *trip)
h.train_step(10)
test = np.random.default_rng(1).integers(0, gr.n_triples, nq)
q = (trip[0][test], trip[1][test], trip[2][test])
filt = kge.filter_lists(trip, *q)
out = {"model": model, "n_entities": gr.n_entities, "dim": 400, "queries": nq,
       "qb": os.environ.get("KGE_RANK_QB", "8"), "split": os.environ.get("KGE_RANK_SPLIT", "auto")}
for name, kw in (("raw", {}), ("filtered", {"filters": filt})):
    h.rank(*q, **kw)
    t0 = time.perf_counter()
    reps = int(os.environ.get("RANK_REPS", "3"))
    for _ in range(reps):
        r = h.rank(*q, **kw)
    dt = (time.perf_counter() - t0) / reps
    out[name] = {"s": dt, "queries_per_s": nq / dt, "scores_per_s": nq * gr.n_entities / dt,
                 "MRR": kge.link_metrics(r)["MRR"]}
print(json.dumps(out))
