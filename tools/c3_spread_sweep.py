"""Pick the C3 mixture spread so the label metrics do not saturate
(cf_10 roughly 0.6-0.9).  For each spread: exact 2-NN graph of
the 1.4M x 100 mixture on the GPU, one 2500-iteration embed, neighbour hit.
Graphs are written to gpurun_out/ (input synthesis, not product)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_05455_b200 import EmbeddingConfig, KnnGraph, run_embedding, metrics, synth

m = int(os.environ.get("M", 1_400_000))
n = int(os.environ.get("N", 100))
c = float(os.environ.get("C", 0.1))
iters = int(os.environ.get("ITERS", 2500))
spreads = [float(s) for s in os.environ.get("SPREADS", "0.25,0.35,0.5,0.7,1.0").split(",")]
os.makedirs("gpurun_out", exist_ok=True)
for sp in spreads:
    t0 = time.perf_counter()
    nb, dist, labels = synth.mixture_knn_graph(m, n, k=2, seed=0, spread=sp)
    tk = time.perf_counter() - t0
    cfg = EmbeddingConfig(nn=2, rn=1, c=c, iterations=iters, seed=0)
    t0 = time.perf_counter()
    res = run_embedding(graph=KnnGraph(nb), config=cfg)
    te = time.perf_counter() - t0
    cf_nn, cf = metrics.neighbor_hit(res.embedding.points, labels, nn_max=100)
    # label agreement of the kNN graph itself (upper reference)
    g_hit = float((labels[nb[:, 0]] == labels).mean())
    print(f"spread {sp}: knn {tk:.1f}s embed {te:.2f}s stress {res.state.stress:.2f} "
          f"cf_2 {cf_nn[1]:.4f} cf_10 {cf_nn[9]:.4f} cf {cf:.4f} graph-nn1-label-agree {g_hit:.4f}", flush=True)
    if os.environ.get("SAVE"):
        np.savez_compressed(f"gpurun_out/graph_m{m}_n{n}_spread{sp}.npz", neighbors=nb)
