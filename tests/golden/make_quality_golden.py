"""Golden end-of-run quality from the REFERENCE on SURVEY §8(d)'s
discriminating C2 fixture: `mnist_like(70000)` -> `pca_reduce(dims=100)` ->
`build_exact_knn(., 2)`, nn=2 rn=1 c=0.01, force-directed, 2500 iterations,
seed 0 (reference: datasets.py:496-553, 289-330; knng.py:158-194;
engine.py:312-414; metrics.py:254-294, 351-380).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_quality_golden.py

Stored (tests/golden/quality_c2.npz): the kNN graph and labels the run used,
the reference's final stress and neighbour-hit curve, and on a fixed 2000-row
subsample (rows `SUB`) the float64 PCA features and the reference's
evaluate_embedding summary of its own embedding.  The GPU test runs the same
graph/config and compares its metrics within 1% (north star).
"""

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "quality_c2.npz")
M, ITERS, N_SUB = 70000, 2500, 2000


def subsample():
    return np.sort(np.random.default_rng(5).choice(M, size=N_SUB, replace=False))


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    from ivhd import datasets, knng, metrics
    from ivhd.engine import EmbeddingConfig, run_embedding

    t = time.time()
    ds = datasets.mnist_like(M, n=784, seed=0)
    red, _ = datasets.pca_reduce(ds, dims=100)
    X = np.asarray(red.data, dtype=np.float64)
    labels = np.asarray(ds.labels)
    g = knng.build_exact_knn(X, 2)
    print("data+knn", time.time() - t, flush=True)
    t = time.time()
    res = run_embedding(graph=g, config=EmbeddingConfig(nn=2, rn=1, c=0.01, iterations=ITERS, seed=0))
    print("run", time.time() - t, flush=True)
    Y = res.embedding.points
    cf_nn, cf = metrics.neighbor_hit(Y, labels, nn_max=100)
    sub = subsample()
    cur = metrics.evaluate_embedding(X[sub], Y[sub], labels=labels[sub], report_ks=(15, 100))
    s = cur.summary()
    print("stress", res.state.stress, "cf", cf, cf_nn[1], cf_nn[9], s, flush=True)
    np.savez_compressed(OUT, neighbors=g.neighbors.astype(np.int32), labels=labels.astype(np.int16),
                        stress=np.float64(res.state.stress), cf_nn=cf_nn, x_sub=X[sub],
                        auc_rnx=np.float64(s["auc_rnx"]), auc_gnn=np.float64(s["auc_gnn"]),
                        trust=np.array([s["trustworthiness_k15"], s["trustworthiness_k100"]]),
                        continuity=np.array([s["continuity_k15"], s["continuity_k100"]]))


if __name__ == "__main__":
    main()
