"""Is the device path host-bound? Host wall time of enqueueing n steps (no sync) vs device time of the same steps."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2004_08532_b200 import kge
gr = synth.graph(sys.argv[1] if len(sys.argv) > 1 else "freebase")
h_, r_, t_ = gr.triples()
cfg = kge.Config(model="transe_l2", n_entities=gr.n_entities, n_relations=gr.n_relations, dim=400, batch_size=1024,
                 chunk_size=256, neg_k=256, neg_precision="tf32")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    H = kge.init(cfg, h_, r_, t_, stream=s)
H.train_step(64, return_loss=False)
H.sync()
for n in (64, 128, 256, 1024, 4096):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    H.sync()
    # hold the device back for a while so the host's enqueue rate is measured unthrottled
    with torch.cuda.stream(s):
        torch.cuda._sleep(int(2e9 * 0.002 * n / 64))
    e0.record(s)
    w0 = time.perf_counter()
    H.train_step(n, return_loss=False)
    w1 = time.perf_counter()
    e1.record(s)
    s.synchronize()
    w2 = time.perf_counter()
    print(f"n={n}: host enqueue {1e6*(w1-w0)/n:.1f} us/step, device {1000*e0.elapsed_time(e1)/n:.1f} us/step, "
          f"wall {1e6*(w2-w0)/n:.1f} us/step")
