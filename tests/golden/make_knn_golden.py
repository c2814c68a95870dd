"""Golden kNN graphs from the REFERENCE `ivhd.knng.build_exact_knn`
(knng.py:158-194), for tests/test_gpu_knn.py.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_knn_golden.py

The inputs are regenerated from seeds by `knn_inputs()` (imported by the
test), so only the reference's neighbours and distances are stored.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def knn_inputs():
    """name -> (matrix, k, metric); deterministic (numpy PCG64 seeds)."""
    out = {}
    rng = np.random.default_rng(11)
    centers = 2.0 * rng.standard_normal((10, 100))
    lab = rng.integers(0, 10, size=3000)
    out["mixture100"] = (centers[lab] + rng.standard_normal((3000, 100)), 10, "euclidean")
    # MNIST-shaped width (784 columns: 24 full K chunks + a partial one)
    rng = np.random.default_rng(12)
    base = rng.standard_normal((20, 784))
    lab = rng.integers(0, 20, size=1500)
    out["wide784"] = (base[lab] + 0.7 * rng.standard_normal((1500, 784)), 5, "euclidean")
    # integer lattice: massive exact distance ties -> the (distance, index) rule
    g = np.arange(12, dtype=np.float64)
    lat = np.stack(np.meshgrid(g, g, g, indexing="ij"), axis=-1).reshape(-1, 3)
    perm = np.random.default_rng(13).permutation(len(lat))
    out["lattice_ties"] = (lat[perm], 8, "euclidean")
    # duplicated rows (zero distances) inside a small random cloud
    rng = np.random.default_rng(14)
    x = rng.standard_normal((800, 16))
    x[400:600] = x[0:200]
    out["duplicates"] = (x, 6, "euclidean")
    # cosine metric (knng.py:105-115)
    rng = np.random.default_rng(15)
    out["cosine64"] = (rng.standard_normal((2500, 64)) + 0.5, 7, "cosine")
    # k beyond the tensor-core pass (k + 4 > 32): every row takes the exact scan
    rng = np.random.default_rng(17)
    out["exact_k40"] = (rng.standard_normal((1200, 24)), 40, "euclidean")
    # precomputed square distance matrix (knng.py:175-181) with exact ties
    rng = np.random.default_rng(18)
    pts = rng.integers(0, 6, (700, 3)).astype(np.float64)
    dmat = np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1))
    out["precomputed_ties"] = (dmat, 9, "precomputed")
    # odd width (not a multiple of 8), k = 1
    rng = np.random.default_rng(16)
    out["odd13_k1"] = (rng.uniform(-1, 1, (1000, 13)), 1, "euclidean")
    return out


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    from ivhd import knng

    arrays = {}
    for name, (x, k, metric) in knn_inputs().items():
        g = knng.build_exact_knn(x, k, metric=metric)
        arrays[f"{name}_nbr"] = g.neighbors
        arrays[f"{name}_dist"] = g.distances
        print(name, x.shape, k, metric)
    np.savez_compressed(os.path.join(HERE, "knn_graphs.npz"), **arrays)
    # the reference's IVHG cache writer (knng.py:286-300) on one of the graphs
    x, k, metric = knn_inputs()["cosine64"]
    g = knng.build_exact_knn(x[:300], 4, metric="cosine")
    knng.cache_write(g, os.path.join(HERE, "ref_cache_cosine.ivhg"))
    knng.cache_write(knng.KnnGraph(g.neighbors, None), os.path.join(HERE, "ref_cache_nodist.ivhg"))


if __name__ == "__main__":
    main()
