"""Where does run_embedding's wall time go at C3 (device RNG path)?  Wraps the
DeviceEmbedding methods run_embedding calls with synchronised host timers."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_05455_b200 import EmbeddingConfig, KnnGraph, run_embedding, synth
from paper_2303_05455_b200 import device as D

nb = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                          "c3_graph.npz"))["neighbors"]  # the C3 bench fixture
T = {}
def wrap(cls, name):
    f = getattr(cls, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); T[name] = T.get(name, 0) + time.perf_counter() - t0
        return r
    setattr(cls, name, g)
for n in ("__init__", "set_optimizer", "init_positions", "set_graph_sampled", "run", "positions", "deltas", "close", "stress"):
    if hasattr(D.DeviceEmbedding, n):
        wrap(D.DeviceEmbedding, n)
cfg = EmbeddingConfig(nn=2, rn=1, c=0.1, iterations=2500, seed=0)
pinned = torch.empty(nb.shape, dtype=torch.int32, pin_memory=True).numpy(); pinned[...] = nb
for rep in range(3):
    T.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    run_embedding(graph=KnnGraph(pinned), config=cfg)
    torch.cuda.synchronize(); wall = time.perf_counter() - t0
    print(f"wall {wall*1e3:.1f} ms: " + "  ".join(f"{k}={v*1e3:.2f}" for k, v in T.items()) +
          f"  other={1e3*(wall-sum(T.values())):.2f}", flush=True)
