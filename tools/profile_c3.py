"""ncu driver for the C3 step kernel in steady state: the committed C3 graph,
the bench's setup, `iters` iterations through ivhd_run (CUDA-graph replays
with PDL, as in the timed loop).  Capture a late launch with
--cache-control none so L2 holds the working set as in the timed loop:

    ncu --set full --cache-control none --clock-control none --import-source on \
        -k regex:step_kernel -s 600 -c 1 -o gpurun_out/c3_steady python tools/profile_c3.py 700
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2303_05455_b200.config import resolve_optimizer
from paper_2303_05455_b200.device import DeviceEmbedding
from paper_2303_05455_b200.embed import init_layout, sample_random_neighbors

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 700
wl = sys.argv[2] if len(sys.argv) > 2 else "c3"
nb = np.load(os.path.join(ROOT, "tests", "golden", "c3_graph.npz"))["neighbors"]
m = nb.shape[0]
rng = np.random.default_rng(0)
y0 = init_layout(m, 2, rng)
rn = sample_random_neighbors(m, nb, 1, rng)
dev = DeviceEmbedding(m, 2)
dev.set_optimizer(resolve_optimizer("force-directed", m))
dev.set_positions(y0)
dev.set_graph(0, nb, rn)
st, _, done, div = dev.run(0, "l2", 0.1, iters)
print(done, div, st[-1])
