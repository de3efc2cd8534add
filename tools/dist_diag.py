import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
from paper_2004_08532_b200 import kge
gr = synth.graph("tiny"); trip = gr.triples()
P = int(os.environ.get("P", "2"))
cfg = kge.Config(model="transe_l2", n_entities=gr.n_entities, n_relations=gr.n_relations, dim=32, batch_size=128,
                 chunk_size=32, neg_k=32, neg_precision="fp32")
hs = kge.init_local_group(cfg, P, *trip)
print("connected", flush=True)
for s in range(int(os.environ.get("STEPS", "2"))):
    for w, h in enumerate(hs):
        h.train_step(1, return_loss=False)
        print("enqueued", s, w, flush=True)
for h in hs:
    h.sync()
print("losses", [h.read_losses(0, 2) for h in hs], flush=True)
