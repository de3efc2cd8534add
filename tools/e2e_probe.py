"""Host-side cost of the e2e path: wall time per kge_train_batch_async call (enqueue only) vs per step end to end."""
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
B, n = 1024, 400
pinned = torch.empty((3, n, B), dtype=torch.int64, pin_memory=True)
idx = np.arange(n * B) % gr.n_triples
for a, arr in enumerate((h_, r_, t_)):
    pinned[a].copy_(torch.from_numpy(np.ascontiguousarray(arr[idx]).reshape(n, B)))
loss = torch.zeros(n, dtype=torch.float32, pin_memory=True)
for rep in range(3):
    H.sync()
    enq = []
    w0 = time.perf_counter()
    ph, pr, pt, pl = pinned[0].data_ptr(), pinned[1].data_ptr(), pinned[2].data_ptr(), loss.data_ptr()
    for st in range(n):
        t0 = time.perf_counter()
        o = st * B * 8
        H.train_batch_async_ptr(ph + o, pr + o, pt + o, pl + 4 * st)
        enq.append(time.perf_counter() - t0)
    w1 = time.perf_counter()
    H.sync()
    w2 = time.perf_counter()
    print(f"rep {rep}: enqueue median {1e6*np.median(enq):.1f} us, p90 {1e6*np.percentile(enq,90):.1f} us; "
          f"enqueue loop {1e6*(w1-w0)/n:.1f} us/step; end to end {1e6*(w2-w0)/n:.1f} us/step")
# device-only reference
H.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s); H.train_step(n, return_loss=False); e1.record(s); s.synchronize()
print(f"device train_step: {1000*e0.elapsed_time(e1)/n:.1f} us/step")
# per-kernel device time on the (non-graph) e2e path, profiler on
H.sync()
H.profile_begin()
for st in range(100):
    H.train_batch_async_ptr(pinned[0, st].data_ptr(), pinned[1, st].data_ptr(), pinned[2, st].data_ptr(), loss[st:].data_ptr())
prof = H.profile_end()
print("profiled e2e path (no graphs):", {k: (round(1000 * v[0], 2), v[1]) for k, v in prof.items() if v[1]})
H.sync()
w0 = time.perf_counter()
for st in range(n):
    H.train_batch_async_ptr(pinned[0, st].data_ptr(), pinned[1, st].data_ptr(), pinned[2, st].data_ptr(), 0)
H.sync()
print(f"no loss readback: {1e6*(time.perf_counter()-w0)/n:.1f} us/step")
