"""Phase timing of k_sample CTAs (KGE_TRACE=1): the ring launch (64 steps) and single-step caller-batch samples."""
import ctypes, os, sys
os.environ["KGE_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2004_08532_b200 import kge
gr = synth.graph(sys.argv[1] if len(sys.argv) > 1 else "freebase")
trip = gr.triples()
cfg = kge.Config(model="transe_l2", n_entities=gr.n_entities, n_relations=gr.n_relations, dim=400, batch_size=1024,
                 chunk_size=256, neg_k=256, neg_precision="tf32")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    h = kge.init(cfg, *trip, stream=s)
L = kge.lib()
L.kge_debug_trace.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int64]
n = 6 * 2048 * 8
def dump(tag):
    buf = np.zeros(n, np.uint64)
    L.kge_debug_trace(h._h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), n)
    T = buf.reshape(6, 2048, 8).astype(np.int64)[0]
    m = T[:, 0] > 0
    T = T[m]
    t0 = T[:, 0].min()
    R = (T - t0) / 1e3
    print(tag, f"ctas={m.sum()}", " ".join(f"s{j} med/max {np.median(R[:, j]):.2f}/{R[:, j].max():.2f}" for j in (0, 1, 2, 7)))
    print("   per-CTA durations s0->s1 / s1->s2 / s2->s7 (med):", np.median(R[:, 1] - R[:, 0]), np.median(R[:, 2] - R[:, 1]), np.median(R[:, 7] - R[:, 2]))
h.train_step(1, return_loss=False); h.sync(); dump("ring (64 steps):")
idx = np.arange(1024)
for k in range(3):
    h.train_batch(trip[0][idx], trip[1][idx], trip[2][idx])
h.sync(); dump("single-step batch:")
