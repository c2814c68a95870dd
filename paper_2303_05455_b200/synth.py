"""Synthetic inputs of the BASELINE.json shapes (input synthesis only — graph
construction is excluded from every timing, as in the paper).

* `planted_graph`  — the SURVEY appendix's locality-friendly kNN-shaped graph
  (10 contiguous clusters, neighbours at small ring offsets).  numpy, O(M k).
* `mixture_knn_graph` — exact kNN graph of a 10-cluster Gaussian mixture in
  N dimensions (the "YAHOO-shaped" 1.4M x 100 input of config C3).  Built on
  the GPU by the package's exact kNN builder (knng.py, csrc/ivhd_knn.cu);
  ids are shuffled like real data, so the graph has realistic hubness and no
  id locality.
"""

import numpy as np


def planted_graph(m, k, seed=0, clusters=10, span=63):
    rng = np.random.default_rng(seed)
    size = max(1, m // clusters)
    ids = np.arange(m)
    cl = np.minimum(ids // size, clusters - 1)
    base = cl * size
    csize = np.where(cl == clusters - 1, m - (clusters - 1) * size, size)
    off = rng.integers(1, span + 1, size=(m, k))
    nb = (ids[:, None] - base[:, None] + off) % csize[:, None] + base[:, None]
    # re-draw duplicates within a row deterministically (next id in the cluster)
    for c in range(1, k):
        dup = (nb[:, c:c + 1] == nb[:, :c]).any(axis=1)
        while dup.any():
            nb[dup, c] = (nb[dup, c] - base[dup] + 1) % csize[dup] + base[dup]
            dup = (nb[:, c:c + 1] == nb[:, :c]).any(axis=1)
    return nb.astype(np.int32)


def mixture_points(m, n, clusters=10, seed=0, spread=2.0):
    """Gaussian mixture, labels = cluster, rows in random order."""
    rng = np.random.default_rng(seed)
    centers = spread * rng.standard_normal((clusters, n)).astype(np.float32)
    labels = rng.integers(0, clusters, size=m)
    x = centers[labels] + rng.standard_normal((m, n), dtype=np.float32)
    return x, labels


def mixture_labels(m, n, clusters=10, seed=0, spread=2.0):
    """The labels of `mixture_points` without drawing the points (same stream)."""
    rng = np.random.default_rng(seed)
    rng.standard_normal((clusters, n)).astype(np.float32)
    return rng.integers(0, clusters, size=m)


def mixture_knn_graph(m, n=100, k=2, clusters=10, seed=0, device=0, block=None, spread=2.0):
    """Exact kNN graph of `mixture_points`, built by this package's GPU kNN
    builder (knng.build_exact_knn: tcgen05 candidate pass + fp64 re-rank).
    Returns (neighbors (m,k) int32, distances (m,k) float64, labels)."""
    from . import knng

    if isinstance(device, str):
        device = int(device.split(":")[1]) if ":" in device else 0
    x, labels = mixture_points(m, n, clusters, seed, spread)
    g = knng.build_exact_knn(x.astype(np.float64), k, device=device)
    return g.neighbors, g.distances, labels
