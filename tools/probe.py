"""Run the diagnostic probe kernels (ivhd_probe) on the C3 graph."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_05455_b200 import synth
from paper_2303_05455_b200.config import resolve_optimizer
from paper_2303_05455_b200.device import DeviceEmbedding
from paper_2303_05455_b200.embed import init_layout, sample_random_neighbors
kind = sys.argv[1] if len(sys.argv) > 1 else "mixture"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1_400_000
cache = f"/tmp/ivhd_graph_mixture_{m}_100_2.npy"
if kind == "mixture":
    nb = np.load(cache) if os.path.exists(cache) else synth.mixture_knn_graph(m, 100, k=2, seed=0)[0]
else:
    nb = synth.planted_graph(m, 2, seed=0)
rng = np.random.default_rng(0)
y0 = init_layout(m, 2, rng); rn = sample_random_neighbors(m, nb[:, :2], 1, rng)
dev = DeviceEmbedding(m, 2); dev.set_optimizer(resolve_optimizer("force-directed", m)); dev.set_positions(y0); dev.set_graph(0, nb[:, :2], rn)
lib = dev.lib
lib.ivhd_probe.restype = ctypes.c_int
lib.ivhd_probe.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
for bps in (4, 8, 16):
    res = []
    for mode in (0, 1, 2):
        us = ctypes.c_double()
        rc = lib.ivhd_probe(dev.h, 0, mode, 50, bps, ctypes.byref(us))
        res.append(f"mode{mode}={us.value:7.2f}us")
    print(kind, m, f"blocks/SM={bps}", " ".join(res), flush=True)
