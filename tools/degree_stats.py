"""Symmetrised-degree statistics of the synthetic workloads (input analysis)."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_05455_b200 import synth

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1_400_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
t = time.time()
nb, _, _ = synth.mixture_knn_graph(m, 100, k=k, seed=0)
print("graph", time.time() - t)
deg = np.bincount(nb.ravel(), minlength=m) + k + 1 + 1  # in-nn + out nn + out rn + ~1 in-rn
q = np.percentile(deg, [50, 90, 99, 99.9, 99.99])
print("deg p50/p90/p99/p99.9/p99.99", q, "max", deg.max(), "mean", deg.mean())
for T in (16, 32, 64, 128, 256, 1024):
    sel = deg > T
    print(f"deg>{T}: vertices {sel.sum()} entries {deg[sel].sum()} ({deg[sel].sum()/deg.sum():.3%})")
np.save("gpurun_out/deg_hist.npy", np.bincount(np.minimum(deg, 100000)))
