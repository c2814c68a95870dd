"""C2 Nesterov on the synthetic MNIST-width mixture: the default alpha (0.02)
diverges in the reference algorithm too (oracle, fp64, iteration 74); find the
largest stable alpha for the bench workload."""
import sys, numpy as np
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
from paper_2303_05455_b200 import synth, EmbeddingConfig, KnnGraph, run_embedding, OptimizerParams
from paper_2303_05455_b200.errors import NumericalDivergenceError
nb, _, _ = synth.mixture_knn_graph(70000, 784, k=5, seed=0)
for a in (0.02, 0.001, 5e-4, 2e-4, 1e-4):
    cfg = EmbeddingConfig(nn=5, rn=1, c=0.01, iterations=2500, seed=0, optimizer="nesterov",
                          opt=OptimizerParams(alpha=a))
    try:
        r = run_embedding(graph=KnnGraph(nb), config=cfg); print(a, "ok", r.trace.stress[-1], flush=True)
    except NumericalDivergenceError as e:
        print(a, "diverged at", e.iteration, flush=True)
