"""Tiny driver for ncu captures: build a graph, run N iterations.
    python tools/profile_one.py planted 10000000 20"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_05455_b200 import synth
from paper_2303_05455_b200.config import resolve_optimizer
from paper_2303_05455_b200.device import DeviceEmbedding
from paper_2303_05455_b200.embed import init_layout, sample_random_neighbors

kind, m, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
nb = synth.planted_graph(m, 2, seed=0) if kind == "planted" else synth.mixture_knn_graph(m, 100, k=2, seed=0)[0]
rng = np.random.default_rng(0)
y0 = init_layout(m, 2, rng)
rn = sample_random_neighbors(m, nb[:, :2], 1, rng)
dev = DeviceEmbedding(m, 2)
dev.set_optimizer(resolve_optimizer("force-directed", m))
dev.set_positions(y0)
dev.set_graph(0, nb[:, :2], rn)
print(dev.run(0, "l2", 0.1, iters)[0][-1])
