"""Synthetic inputs of the BASELINE.json shapes (input synthesis only — graph
construction is excluded from every timing, as in the paper).

* `planted_graph`  — the SURVEY appendix's locality-friendly kNN-shaped graph
  (10 contiguous clusters, neighbours at small ring offsets).  numpy, O(M k).
* `mixture_knn_graph` — exact kNN graph of a 10-cluster Gaussian mixture in
  N dimensions (the "YAHOO-shaped" 1.4M x 100 input of config C3).  Built on
  the GPU by blocked brute force with torch (setup plumbing: matmul + topk);
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


def mixture_knn_graph(m, n=100, k=2, clusters=10, seed=0, device="cuda", block=4096):
    """Brute-force (TF32) kNN of `mixture_points` on the GPU.  Returns
    (neighbors (m,k) int32, distances (m,k) float64, labels)."""
    import torch

    x, labels = mixture_points(m, n, clusters, seed)
    X = torch.from_numpy(x).to(device)
    sq = (X * X).sum(dim=1)
    nbr = torch.empty((m, k), dtype=torch.int64, device=device)
    dst = torch.empty((m, k), dtype=torch.float32, device=device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True  # input synthesis: speed over exact ties
    try:
        for s in range(0, m, block):
            e = min(s + block, m)
            d2 = sq[s:e, None] + sq[None, :] - 2.0 * (X[s:e] @ X.T)
            d2[torch.arange(e - s, device=device), torch.arange(s, e, device=device)] = float("inf")
            v, i = torch.topk(d2, k, dim=1, largest=False, sorted=True)
            nbr[s:e] = i
            dst[s:e] = v.clamp_min(0).sqrt()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return (nbr.cpu().numpy().astype(np.int32), dst.cpu().numpy().astype(np.float64), labels)
