"""Inputs and REFERENCE results for the small BASELINE configs.

C1 (configs[0]): 20k x 784 ten-cluster Gaussian mixture
    `synth.mixture_points(20000, 784, seed=0, spread=C1_SPREAD)` (spread chosen
    so the label metrics do not saturate, tools/c3_spread_sweep.py), exact 2-NN
    graph by the reference's `knng.build_exact_knn`, nn=2 rn=1 c=0.01,
    force-directed, 2000 iterations, seed 0.
C2 (configs[1]): the reference's `datasets.mnist_like(70000, 784, seed=0)`
    (datasets.py:496-553), exact 5-NN graph by `build_exact_knn`, nn=5 rn=1
    c=0.01, 2500 iterations, Adadelta and Nesterov at their default alpha.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_c1c2_golden.py

Writes tests/golden/c1_golden.npz and tests/golden/c2_golden.npz: the graph
(int32) and labels (the bench's inputs: nothing here needs the reference or
the data at run time), and the reference's own full-run results —
engine.run_embedding (engine.py:312-414) final stress, stress/b traces,
metrics.neighbor_hit (metrics.py:254-294) and, for C1, the
metrics.evaluate_embedding summary over all 20k rows (metrics.py:355-385).
"""

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
C1_SPREAD = float(os.environ.get("C1_SPREAD", "0.23"))


def run(graph, labels, **cfg):
    from ivhd import metrics
    from ivhd.engine import EmbeddingConfig, run_embedding

    t = time.time()
    res = run_embedding(graph=graph, config=EmbeddingConfig(seed=0, **cfg), threads=os.cpu_count() or 1)
    cf_nn, cf = metrics.neighbor_hit(res.embedding.points, labels, nn_max=100)
    print(cfg, "run+hit", round(time.time() - t, 1), "s stress", res.state.stress, "cf", cf, flush=True)
    return res, cf_nn, cf


def main(which):
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    sys.path.insert(0, ROOT)
    from ivhd import datasets, knng, metrics

    from paper_2303_05455_b200 import synth

    if "c1" in which:
        x, labels = synth.mixture_points(20000, 784, seed=0, spread=C1_SPREAD)
        xd = x.astype(np.float64)
        t = time.time()
        g = knng.build_exact_knn(xd, 2)
        print("c1 knn", time.time() - t, flush=True)
        res, cf_nn, cf = run(g, labels, nn=2, rn=1, c=0.01, iterations=2000)
        t = time.time()
        s = metrics.evaluate_embedding(xd, res.embedding.points, labels=labels, nn_max=100,
                                       report_ks=(15, 100)).summary()
        print("c1 curves", time.time() - t, s, flush=True)
        np.savez_compressed(
            os.path.join(HERE, "c1_golden.npz"), neighbors=g.neighbors.astype(np.int32),
            labels=labels.astype(np.int8), spread=np.float64(C1_SPREAD), stress=np.float64(res.state.stress),
            trace_stress=np.asarray(res.trace.stress), trace_b=np.asarray(res.trace.step_size),
            cf_nn=cf_nn, cf=np.float64(cf), summary_keys=np.array(sorted(s)),
            summary_vals=np.array([float(s[k]) for k in sorted(s)]))
    if "c2" in which:
        t = time.time()
        ds = datasets.mnist_like(70000, n=784, seed=0)
        labels = np.asarray(ds.labels)
        g = knng.build_exact_knn(np.asarray(ds.data, dtype=np.float64), 5)
        print("c2 data+knn", time.time() - t, flush=True)
        out = {"neighbors": g.neighbors.astype(np.int32), "labels": labels.astype(np.int8)}
        for opt in ("adadelta", "nesterov"):
            res, cf_nn, cf = run(g, labels, nn=5, rn=1, c=0.01, iterations=2500, optimizer=opt)
            out.update({f"{opt}_stress": np.float64(res.state.stress),
                        f"{opt}_trace_stress": np.asarray(res.trace.stress),
                        f"{opt}_trace_b": np.asarray(res.trace.step_size),
                        f"{opt}_cf_nn": cf_nn, f"{opt}_cf": np.float64(cf)})
        np.savez_compressed(os.path.join(HERE, "c2_golden.npz"), **out)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2"])
