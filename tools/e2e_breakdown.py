"""Where does run_embedding's wall time go at C3 (1.4M)?  Times each phase of
the public path with host timers (device synchronised)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_05455_b200 import EmbeddingConfig, KnnGraph, run_embedding, synth
from paper_2303_05455_b200.config import resolve_optimizer
from paper_2303_05455_b200.device import DeviceEmbedding
from paper_2303_05455_b200.embed import init_layout, sample_random_neighbors

cache = "/tmp/ivhd_graph_mixture_1400000_100_2.npy"
nb = np.load(cache) if os.path.exists(cache) else synth.mixture_knn_graph(1_400_000, 100, k=2, seed=0)[0]
m = nb.shape[0]
T = {}
def tick(name, t0):
    torch.cuda.synchronize(); T[name] = T.get(name, 0) + time.perf_counter() - t0; return time.perf_counter()
for rep in range(2):
    T.clear()
    t = time.perf_counter()
    rng = np.random.default_rng(0)
    y0 = init_layout(m, 2, rng); t = tick("init_layout", t)
    rn = sample_random_neighbors(m, nb[:, :2], 1, rng); t = tick("sample_rn", t)
    dev = DeviceEmbedding(m, 2); t = tick("ctx_create", t)
    dev.set_optimizer(resolve_optimizer("force-directed", m)); t = tick("set_optimizer", t)
    dev.set_positions(y0); t = tick("set_positions", t)
    dev.set_graph(0, nb[:, :2], rn); t = tick("set_graph(csr+relabel)", t)
    dev.run(0, "l2", 0.1, 2500); t = tick("run_2500", t)
    p = dev.positions(); t = tick("positions", t)
    d = dev.deltas(); t = tick("deltas", t)
    dev.close(); t = tick("close", t)
    tot = sum(T.values())
    print(f"rep {rep}: total {tot*1e3:.1f} ms  " + "  ".join(f"{k}={v*1e3:.1f}" for k, v in T.items()))
cfg = EmbeddingConfig(nn=2, rn=1, c=0.1, iterations=2500, seed=0)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    run_embedding(graph=KnnGraph(nb), config=cfg)
    torch.cuda.synchronize(); print(f"run_embedding wall {1e3*(time.perf_counter()-t0):.1f} ms")
