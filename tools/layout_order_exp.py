"""Experiment: how much would a layout-driven vertex order speed up the C3
loop?  Runs the C3 embed for R iterations, orders the vertices along a
Hilbert curve of the current 2-D layout, relabels the graph (nn ids and the
same rn partners) on the host, and times the steady-state loop on the
original and the relabelled graph from the same positions.  (Experiment
only: the product does this on the device, ivhd_capi.cu relayout.)"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2303_05455_b200 import EmbeddingConfig, KnnGraph, run_embedding
from paper_2303_05455_b200.config import resolve_optimizer
from paper_2303_05455_b200.device import DeviceEmbedding


def hilbert_keys(y, bits=16):
    """Hilbert index of the layout quantised to 2^bits x 2^bits (xy2d)."""
    n = 1 << bits
    lo, hi = y.min(axis=0), y.max(axis=0)
    q = ((y - lo) / np.maximum(hi - lo, 1e-30) * (n - 1)).astype(np.int64)
    x, yy = q[:, 0].copy(), q[:, 1].copy()
    d = np.zeros(len(q), dtype=np.int64)
    s = n >> 1
    while s > 0:
        rx = ((x & s) > 0).astype(np.int64)
        ry = ((yy & s) > 0).astype(np.int64)
        d += s * s * ((3 * rx) ^ ry)
        flip = (ry == 0) & (rx == 1)
        x = np.where(flip, n - 1 - x, x)
        yy = np.where(flip, n - 1 - yy, yy)
        sw = ry == 0
        x, yy = np.where(sw, yy, x), np.where(sw, x, yy)
        s >>= 1
    return d


def timed_loop(nb, rn, y, iters=500, reps=3):
    m = nb.shape[0]
    dev = DeviceEmbedding(m, 2)
    dev.set_optimizer(resolve_optimizer("force-directed", m))
    dev.set_positions(y)
    dev.set_graph(0, nb, rn)
    dev.snapshot()
    best = 1e9
    for _ in range(reps + 1):
        dev.restore()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.run(0, "l2", 0.1, iters)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    out = dev.positions()
    dev.close()
    return best / iters * 1e6, out


def main():
    nb = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c3_graph.npz"))["neighbors"]
    m = nb.shape[0]
    for R in [int(r) for r in os.environ.get("R", "100,500,2500").split(",")]:
        res = run_embedding(graph=KnnGraph(nb), config=EmbeddingConfig(nn=2, rn=1, c=0.1, iterations=R, seed=0))
        y, rn = res.embedding.points, res.state.rn_assignments
        t_orig, _ = timed_loop(nb, rn, y)
        order = np.argsort(hilbert_keys(y), kind="stable")  # new -> old
        inv = np.empty(m, dtype=np.int64)
        inv[order] = np.arange(m)
        nb2 = inv[nb[order]].astype(np.int32)
        rn2 = inv[rn[order]].astype(np.int32)
        t_hil, y2 = timed_loop(nb2, rn2, y[order])
        local = np.mean(np.abs(nb2 - np.arange(m)[:, None]) < 2048)
        print(f"R={R}: original order {t_orig:.1f} us/it, hilbert-relabelled {t_hil:.1f} us/it "
              f"(nn partners within 2048 ids: {local:.3f})", flush=True)


if __name__ == "__main__":
    main()
