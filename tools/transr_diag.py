import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O, synth
from paper_2004_08532_b200 import kge
gr = synth.graph("tiny"); trip = gr.triples()
B, g, k, d = 64, 16, 16, 32
MODEL = os.environ.get("MODEL", "transr")
print("init", flush=True)
cfg = kge.Config(model=MODEL, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=d, batch_size=B, chunk_size=g,
                 neg_k=k, lr=0.05, neg_precision="fp32")
h = kge.init(cfg, *trip)
print("score", flush=True)
print(h.score([0, 1], [0, 1], [2, 3]), flush=True)
orc = O.Trainer(MODEL, gr.n_entities, gr.n_relations, d, B, g, k, lr=0.05, triples=trip)
print("oracle score", orc.score_triples([0, 1], [0, 1], [2, 3]), flush=True)
print("train 1", flush=True)
t = time.time(); l = h.train_step(1); print("gpu loss", l, time.time() - t, flush=True)
t = time.time(); lo = orc.train(1); print("orc loss", lo, time.time() - t, flush=True)
