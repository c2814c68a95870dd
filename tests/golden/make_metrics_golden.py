"""Golden neighbour-hit values from the REFERENCE `ivhd.metrics.neighbor_hit`
(metrics.py:254-294), for tests/test_gpu_metrics.py.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_metrics_golden.py

Inputs are regenerated from seeds by `metric_inputs()`; only the reference's
cf_nn curves are stored.  Sizes cover both reference branches: M <= 20000
(exact build_exact_knn) and M > 20000 in 2-D (cKDTree).
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def metric_inputs():
    out = {}
    rng = np.random.default_rng(21)
    c = rng.uniform(-5, 5, (8, 2))
    lab = rng.integers(0, 8, 4000)
    out["blobs2d_4k"] = (c[lab] + rng.standard_normal((4000, 2)), lab, 100)
    rng = np.random.default_rng(22)
    c = rng.uniform(-3, 3, (10, 2))
    lab = rng.integers(0, 10, 30000)
    out["blobs2d_30k"] = (c[lab] + 0.8 * rng.standard_normal((30000, 2)), lab, 100)
    rng = np.random.default_rng(23)
    c = rng.uniform(-3, 3, (5, 3))
    lab = rng.integers(0, 5, 5000)
    out["blobs3d_5k_k30"] = (c[lab] + rng.standard_normal((5000, 3)), lab, 30)
    # integer grid: exact distance ties everywhere (index tie rule)
    g = np.arange(60, dtype=np.float64)
    pts = np.stack(np.meshgrid(g, g, indexing="ij"), -1).reshape(-1, 2)
    lab = ((pts[:, 0] // 7 + pts[:, 1] // 5) % 3).astype(np.int64)
    out["grid2d_ties_k12"] = (pts, lab, 12)
    return out


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    from ivhd import metrics

    arrays = {}
    for name, (y, lab, k) in metric_inputs().items():
        cf_nn, cf = metrics.neighbor_hit(y, lab, nn_max=k)
        arrays[name] = cf_nn
        print(name, y.shape, k, cf)
    np.savez_compressed(os.path.join(HERE, "neighbor_hit.npz"), **arrays)


if __name__ == "__main__":
    main()
