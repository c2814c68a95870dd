"""How local are nn partners in a Hilbert order of the current layout?
(Decides whether a layout-driven relabelling can cut the step kernel's
L1->L2 gather requests.)"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from layout_order_exp import hilbert_keys
from paper_2303_05455_b200 import EmbeddingConfig, KnnGraph, run_embedding

nb = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c3_graph.npz"))["neighbors"]
m = nb.shape[0]
for R in (50, 200, 1000, 2500):
    res = run_embedding(graph=KnnGraph(nb), config=EmbeddingConfig(nn=2, rn=1, c=0.1, iterations=R, seed=0))
    y = res.embedding.points
    rank = np.empty(m, dtype=np.int64)
    rank[np.argsort(hilbert_keys(y), kind="stable")] = np.arange(m)
    dr = np.abs(rank[nb] - rank[:, None]).ravel()
    d = np.sqrt(((y[nb] - y[:, None, :]) ** 2).sum(-1)).ravel()
    span = np.ptp(y, axis=0)
    print(f"R={R}: layout span {span.round(2)}, nn distance p50 {np.median(d):.4f} p90 {np.quantile(d, .9):.4f}; "
          "nn partners within Hilbert-rank distance " +
          " ".join(f"{w}:{np.mean(dr < w):.3f}" for w in (256, 1024, 4096, 16384, 65536)), flush=True)
