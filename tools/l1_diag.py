"""Diagnostic: where does the TransE-L1 FP32 trajectory leave the fp64 oracle? (kink flips of sgn(h+r-t))"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import synth
from paper_2004_08532_b200 import kge

gr = synth.graph("tiny")
trip = gr.triples()
for (B, g, k, d) in [(256, 64, 64, 64), (64, 16, 16, 32)]:
    for model in ["transe_l1", "transe_l2"]:
        cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=d, batch_size=B,
                         chunk_size=g, neg_k=k, neg_precision="fp32")
        h = kge.init(cfg, *trip)
        orc = O.Trainer(model, gr.n_entities, gr.n_relations, d, B, g, k, triples=trip)
        lg, lo = h.train_step(100), orc.train(100)
        rel = np.abs(lg - lo) / np.abs(lo)
        first = int(np.argmax(rel > 1e-6)) if (rel > 1e-6).any() else -1
        ids = np.arange(gr.n_entities)
        dE = np.abs(h.get_rows(0, ids) - orc.get_rows(0, ids)).max()
        print(model, (B, g, k, d), "max rel", rel.max(), "first>1e-6 at", first, "rows maxdiff", dE, flush=True)
        # teacher forced: copy oracle tables into the GPU each step
        orc2 = O.Trainer(model, gr.n_entities, gr.n_relations, d, B, g, k, triples=trip)
        h2 = kge.init(cfg, *trip)
        worst = 0.0
        rids = np.arange(gr.n_relations)
        for s in range(30):
            for tab, ids_ in ((0, ids), (1, rids), (3, ids), (4, rids)):
                h2.set_rows(tab, ids_, orc2.get_rows(tab, ids_))
            l1 = h2.train_step(1)[0]
            l2 = orc2.train(1)[0]
            worst = max(worst, np.abs(h2.get_rows(0, ids) - orc2.get_rows(0, ids)).max())
        print("  teacher-forced 30 steps: worst row diff", worst, flush=True)
