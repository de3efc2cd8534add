import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2004_08532_b200 import kge
gr = synth.graph("tiny"); trip = gr.triples()
model, B, g, k, d = sys.argv[1], *map(int, sys.argv[2:6])
cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=d, batch_size=B, chunk_size=g,
                 neg_k=k, neg_precision="fp32")
h = kge.init(cfg, *trip)
print(model, B, g, k, d, h.train_step(2), flush=True)
