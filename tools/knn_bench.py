"""Time the GPU kNN builder on the C3 shape (YAHOO-shaped 10-cluster mixture,
M x 100) and check sampled rows against an fp64 torch scan.
    python tools/knn_bench.py [M] [k]"""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_05455_b200 import knng, synth

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1_400_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
x, labels = synth.mixture_points(m, 100, seed=0)
x = x.astype(np.float64)
knng.build_exact_knn(x[:4096], k)  # warm-up (module load, context)
t0 = time.perf_counter()
g = knng.build_exact_knn(x, k)
wall = time.perf_counter() - t0
out = dict(m=m, n=100, k=k, wall_s=wall, **knng.last_stats)
import torch
X = torch.from_numpy(x).cuda()
rng = np.random.default_rng(1)
rows = rng.choice(m, 64, replace=False)
d = torch.cdist(X[rows], X).cpu().numpy()
d[np.arange(64), rows] = np.inf
ok = 0
for i, r in enumerate(rows):
    order = np.lexsort((np.arange(m), d[i]))[:k]
    ok += int((g.neighbors[r] == order).all())
out["sampled_rows_exact"] = f"{ok}/64"
tc_flops = 2.0 * m * m * 104
out["tc_tflops"] = tc_flops / out["tc_seconds"] / 1e12
print(json.dumps(out))
