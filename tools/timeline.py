"""Per-unit phase timeline of the step kernel (debug build with -DIVHD_TIMELINE)."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_05455_b200 import synth
from paper_2303_05455_b200.config import resolve_optimizer
from paper_2303_05455_b200.device import DeviceEmbedding
from paper_2303_05455_b200.embed import init_layout, sample_random_neighbors
cache = "/tmp/ivhd_graph_mixture_1400000_100_2.npy"
nb = np.load(cache) if os.path.exists(cache) else synth.mixture_knn_graph(1_400_000, 100, k=2, seed=0)[0]
m = nb.shape[0]; rng = np.random.default_rng(0)
y0 = init_layout(m, 2, rng); rn = sample_random_neighbors(m, nb[:, :2], 1, rng)
dev = DeviceEmbedding(m, 2); dev.set_optimizer(resolve_optimizer("force-directed", m)); dev.set_positions(y0); dev.set_graph(0, nb[:, :2], rn)
dev.run(0, "l2", 0.1, 20)
lib = ctypes.CDLL(os.environ["IVHD_B200_LIB"])
buf = np.zeros(8 * 64 * 6, np.int64)
lib.ivhd_timeline_dump(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)))
t = buf.reshape(8, 64, 6).astype(np.float64)
for b in range(3):
    base = t[b, 0, 0]
    print(f"block {b}")
    for k in range(16):
        r = t[b, k]
        if r[0] == 0: break
        print(f"  unit {k:2d} start {r[0]-base:8.0f}  producer {r[1]-r[0]:6.0f}  wait-done {r[2]-r[0]:6.0f}  compute {r[3]-r[2]:6.0f}  barrier {r[4]-r[3]:6.0f}  next {t[b,k+1,0]-r[0] if t[b,k+1,0] else 0:6.0f}")
d = t[:, 1:40]
valid = d[:, :, 0] > 0
print("median cycles: producer", np.median((d[:,:,1]-d[:,:,0])[valid]), "wait", np.median((d[:,:,2]-d[:,:,1])[valid]),
      "compute", np.median((d[:,:,3]-d[:,:,2])[valid]), "barrier", np.median((d[:,:,4]-d[:,:,3])[valid]))
