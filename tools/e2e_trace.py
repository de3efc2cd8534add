"""KGE_TRACE timeline of the caller-batch (e2e) path: last step's sample CTAs vs its step kernels."""
import ctypes, os, sys
os.environ["KGE_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2004_08532_b200 import kge
gr = synth.graph("freebase")
h_, r_, t_ = gr.triples()
cfg = kge.Config(model="transe_l2", n_entities=gr.n_entities, n_relations=gr.n_relations, dim=400, batch_size=1024,
                 chunk_size=256, neg_k=256, neg_precision="tf32")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    H = kge.init(cfg, h_, r_, t_, stream=s)
B, n = 1024, 64
pinned = torch.empty((3, n, B), dtype=torch.int64, pin_memory=True)
idx = np.arange(n * B) % gr.n_triples
for a, arr in enumerate((h_, r_, t_)):
    pinned[a].copy_(torch.from_numpy(np.ascontiguousarray(arr[idx]).reshape(n, B)))
loss = torch.zeros(n, dtype=torch.float32, pin_memory=True)
ph, pr, pt, pl = pinned[0].data_ptr(), pinned[1].data_ptr(), pinned[2].data_ptr(), loss.data_ptr()
for st in range(n):
    H.train_batch_async_ptr(ph + st * B * 8, pr + st * B * 8, pt + st * B * 8, pl + 4 * st)
H.sync()
L = kge.lib()
L.kge_debug_trace.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int64]
nn = 6 * 2048 * 8
buf = np.zeros(nn, np.uint64)
L.kge_debug_trace(H._h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), nn)
T = buf.reshape(6, 2048, 8).astype(np.int64)
names = kge.KERNELS
t0 = T[1][:, 0][T[1][:, 0] > 0].min()
for k in range(6):
    m = T[k][:, 0] > 0
    if not m.any():
        continue
    R = (T[k][m] - t0) / 1e3
    ends = R[:, 7][T[k][m][:, 7] > 0]
    print(f"{names[k]:10s} ctas={m.sum():5d} start min/med/max {R[:,0].min():8.2f}/{np.median(R[:,0]):8.2f}/{R[:,0].max():8.2f}"
          f"  s1 med {np.median(R[:,1]):8.2f}  end med/max {np.median(ends) if len(ends) else 0:8.2f}/{ends.max() if len(ends) else 0:8.2f}")
