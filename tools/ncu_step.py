"""Minimal driver for ncu captures: the bench workload (freebase TransE-L2 TF32), N steps, no timing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2004_08532_b200 import kge
wl = sys.argv[1] if len(sys.argv) > 1 else "freebase"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
model = sys.argv[3] if len(sys.argv) > 3 else "transe_l2"
dim = int(sys.argv[4]) if len(sys.argv) > 4 else 400
gr = synth.graph(wl)
cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=dim, batch_size=1024,
                 chunk_size=256, neg_k=256, neg_precision="tf32")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    h = kge.init(cfg, *gr.triples(), stream=s)
h.train_step(steps, return_loss=False)
h.sync()
print("ok")
