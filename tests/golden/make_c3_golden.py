"""Golden full-run result from the REFERENCE at the headline config C3
(BASELINE.json configs[2]): the exact 2-NN graph of the
1.4M x 100 ten-cluster Gaussian mixture `synth.mixture_points(1_400_000, 100,
seed=0, spread=C3_SPREAD)` (spread chosen so the label metrics do not
saturate: cf_10 in 0.6-0.9, tools/c3_spread_sweep.py), nn=2 rn=1 c=0.1,
force-directed with the reference defaults, 2500 iterations, seed 0.

    # 1. on a GPU box: the graph, built by the package's exact kNN builder
    #    (bit-identical to the reference's build_exact_knn, tests/test_gpu_knn.py)
    gpurun -- 'SAVE=1 SPREADS=0.42 python tools/c3_spread_sweep.py'
    # 2. here (the reference is importable only in this container):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_c3_golden.py gpurun_out/c3_graph_spread0.42.npz

The reference (engine.run_embedding, engine.py:312-414, threads = all host
cores; metrics.neighbor_hit, metrics.py:254-294; metrics.evaluate_embedding,
metrics.py:355-385 on a fixed seeded 20k-row subsample) runs in float64 on the
CPU.  Stored in tests/golden/quality_c3.npz (small: no positions, no graph):
the graph's sha256 (the GPU test rebuilds the graph and checks it), the
positions of 4096 fixed rows after each of the first 10 iterations, the
stress / step-size trace of all 2500 iterations, the final stress, the
neighbour-hit curve over all 1.4M points, and the subsample summary.
"""

import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "quality_c3.npz")
M, N, ITERS, N_SUB = 1_400_000, 100, 2500, 20000
C3_SPREAD = 0.42


def subsample():
    return np.sort(np.random.default_rng(0).choice(M, size=N_SUB, replace=False))


def graph_sha(nb):
    return hashlib.sha256(np.ascontiguousarray(nb, dtype=np.int32).tobytes()).hexdigest()


def main(path):
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    sys.path.insert(0, ROOT)
    from ivhd import metrics
    from ivhd.engine import EmbeddingConfig, run_embedding
    from ivhd.knng import KnnGraph

    from paper_2303_05455_b200 import synth

    nb = np.load(path)["neighbors"].astype(np.int32)
    assert nb.shape == (M, 2), nb.shape
    x, labels = synth.mixture_points(M, N, seed=0, spread=C3_SPREAD)
    # the graph really is the exact 2-NN graph of these points (spot check, fp64)
    rows = np.random.default_rng(1).choice(M, size=8, replace=False)
    xd = x.astype(np.float64)
    for r in rows:
        d = ((xd - xd[r]) ** 2).sum(axis=1)
        d[r] = np.inf
        best = np.lexsort((np.arange(M), d))[:2]
        assert (best == nb[r]).all(), (r, best, nb[r])
    g = KnnGraph(neighbors=nb, distances=np.zeros(nb.shape), metric="euclidean")
    t = time.time()
    trace = []
    rows10 = np.sort(np.random.default_rng(2).choice(M, size=4096, replace=False))
    early = []

    def observer(it, positions, stress, params):
        trace.append((stress, params["b"]))
        if it < 10:  # positions after iterations 1..10 on a fixed row sample
            early.append(np.array(positions[rows10]))
        if it % 100 == 0:
            print(f"it {it} stress {stress:.6f} b {params['b']} {time.time() - t:.0f}s", flush=True)
        return None

    threads = os.cpu_count() or 1
    res = run_embedding(graph=g, config=EmbeddingConfig(nn=2, rn=1, c=0.1, iterations=ITERS, seed=0),
                        observer=observer, threads=threads)
    print("run", time.time() - t, "s", flush=True)
    Y = res.embedding.points
    t = time.time()
    cf_nn, cf = metrics.neighbor_hit(Y, labels, nn_max=100)
    print("neighbor_hit", time.time() - t, cf, cf_nn[1], cf_nn[9], flush=True)
    sub = subsample()
    t = time.time()
    cur = metrics.evaluate_embedding(xd[sub], Y[sub], labels=labels[sub], nn_max=100, report_ks=(15, 100))
    s = cur.summary()
    print("curves", time.time() - t, s, flush=True)
    tr = np.array(trace)
    np.savez_compressed(
        OUT, graph_sha256=np.array(graph_sha(nb)), spread=np.float64(C3_SPREAD),
        trace_stress=tr[:, 0], trace_b=tr[:, 1], stress=np.float64(res.state.stress),
        stress_trace_engine=np.asarray(res.trace.stress), b_trace_engine=np.asarray(res.trace.step_size),
        cf_nn=cf_nn, cf=np.float64(cf), sub=sub.astype(np.int32),
        auc_rnx=np.float64(s["auc_rnx"]), auc_gnn=np.float64(s["auc_gnn"]),
        summary_keys=np.array(sorted(s)), summary_vals=np.array([float(s[k]) for k in sorted(s)]),
        threads=np.int64(threads), rows10=rows10.astype(np.int32), early_positions=np.stack(early))
    print("wrote", OUT)


if __name__ == "__main__":
    main(sys.argv[1])
