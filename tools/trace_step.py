"""Per-CTA timeline of one training step (KGE_TRACE=1): kernel spans, CTA start spread, TC phases."""
import ctypes, os, sys
os.environ["KGE_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2004_08532_b200 import kge
wl = sys.argv[1] if len(sys.argv) > 1 else "freebase"
ov = {}
if os.environ.get("KGE_TRACE_NE"):  # experiments: a smaller entity table (and triple list) of the same shape
    ov = dict(n_entities=int(os.environ["KGE_TRACE_NE"]), n_triples=int(os.environ.get("KGE_TRACE_NT", 20_000_000)))
gr = synth.graph(wl, **ov)
trip = gr.triples()
cfg = kge.Config(model="transe_l2", n_entities=gr.n_entities, n_relations=gr.n_relations, dim=400, batch_size=1024,
                 chunk_size=256, neg_k=256, neg_precision="tf32")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    h = kge.init(cfg, *trip, stream=s)
steady = "steady" in sys.argv  # steady: the traced step is the last of a back-to-back run (host far ahead)
prof = "prof" in sys.argv  # the bench's isolated-kernel mode: profiler on (events around launches, PDL off)
if steady:
    h.train_step(71, return_loss=False)
else:
    h.train_step(70, return_loss=False)
    h.sync()
    if prof:
        h.profile_begin()
    h.train_step(1, return_loss=False)
    if prof:
        print("profile (ms):", {k: round(v[0], 4) for k, v in h.profile_end().items() if v[1]})
h.sync()
L = kge.lib()
L.kge_debug_trace.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int64]
n = 6 * 2048 * 8
buf = np.zeros(n, np.uint64)
L.kge_debug_trace(h._h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), n)
T = buf.reshape(6, 2048, 8).astype(np.int64)
names = kge.KERNELS
t0 = min(T[k][:, 0][T[k][:, 0] > 0].min() for k in range(1, 6) if (T[k][:, 0] > 0).any())
for k in range(1, 6):
    st = T[k][:, 0]
    m = st > 0
    if not m.any():
        continue
    st = st[m] - t0
    en = T[k][:, 7][m]
    en = en[en > 0] - t0 if (en > 0).any() else np.array([0])
    line = f"{names[k]:10s} ctas={m.sum():5d} start[min/med/max]={st.min()/1e3:6.2f}/{np.median(st)/1e3:6.2f}/{st.max()/1e3:6.2f} us  end med/max={np.median(en)/1e3:6.2f}/{en.max()/1e3:6.2f} us"
    if k in (1, 5):
        w6 = T[k][:, 6][m]
        w6 = w6[w6 > 0]
        if len(w6):
            line += f" | last warp end {(w6.max() - t0)/1e3:6.2f}"
    r1 = T[k][:, 1][m]
    r1 = r1[r1 > 0]
    if len(r1):
        line += f" | released(s1) min/med {(r1.min() - t0)/1e3:6.2f}/{(np.median(r1) - t0)/1e3:6.2f}"
    if k == 1 and (T[k][:, 1][m] > 0).any():
        s1 = T[k][:, 1][m]
        s1 = s1[s1 > 0] - t0
        line += f" | after pdl_wait min/med/max {s1.min()/1e3:6.2f}/{np.median(s1)/1e3:6.2f}/{s1.max()/1e3:6.2f}"
        if T[k][0, 2] > 0:
            line += f" | prev update end {(int(T[k][0, 2]) - t0)/1e3:6.2f}"
            line += f", last start {(int(T[k][0, 3]) - t0)/1e3:6.2f}"
    if k in (2, 3):
        s1 = T[k][:, 1][m] - t0
        s2 = T[k][:, 2][m] - t0
        s2 = s2[T[k][:, 2][m] > 0]
        line += f" | setup done med {np.median(s1)/1e3:6.2f}, mainloop done med/max {np.median(s2)/1e3:6.2f}/{s2.max()/1e3:6.2f}"
        for sl in (3, 4, 5, 6):
            x = T[k][:, sl][m]
            x = x[x > 0] - t0
            if len(x):
                line += f" | s{sl} med {np.median(x)/1e3:6.2f}"
    print(line)
# backward split by pass (z = 0: dO / fused chain, z = 1: dX'); CTAs are numbered x + gx*(y + gy*z)
k = 3
m = T[k][:, 0] > 0
n = m.sum()
for z, sl in ((0, slice(0, n // 2)), (1, slice(n // 2, n))):
    R = T[k][:n][sl] - t0
    cols = " ".join(f"s{j} {np.median(R[:, j])/1e3:6.2f}/{R[:, j].max()/1e3:6.2f}" for j in range(8))
    print(f"  bwd z={z}: med/max {cols}")
# update: entity CTAs first (n_occ / 8 of them), then one CTA per unique relation
k = 5
U = T[k]
nr = 1024 // 8  # warp per segment start: relation positions first (B / 8 CTAs), then the entity positions
for name, sl in (("relation", slice(0, nr)), ("entity", slice(nr, 2048))):
    R = U[sl]
    m = R[:, 7] > 0
    if not m.any():
        continue
    R = R[m] - t0
    cols = " ".join(f"s{j} {np.median(R[:, j])/1e3:6.2f}/{R[:, j].max()/1e3:6.2f}" for j in (0, 1, 2, 3, 7) if (U[sl][m][:, j] > 0).all())
    print(f"  update {name:8s} n={m.sum():4d}: med/max {cols}")
