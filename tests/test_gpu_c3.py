"""Parity at the headline configurations.

C3 (BASELINE.json configs[2]): the exact 2-NN graph of the non-saturating
1.4M x 100 mixture (spread 0.42: cf_10 ~ 0.76), nn=2 rn=1 c=0.1,
force-directed, seed 0.  The golden file tests/golden/quality_c3.npz was made
by the REFERENCE itself (tests/golden/make_c3_golden.py: ivhd.engine.run_embedding
in float64 on the CPU, 2500 iterations, plus its metrics), so these tests
compare the CUDA path directly with the reference at full size:

* the graph the GPU builds is the golden run's input (sha256);
* 10 iterations: positions of 4096 fixed rows after every iteration within
  1e-5 normwise, stress within 1e-5, the step-size trace exact; forces at
  the final positions within 1e-5 of the oracle (numpy restatement, pinned
  to the reference by tests/test_oracle_golden.py);
* the full 2500-iteration embed: final stress, the whole b trace, the
  neighbour-hit curve over all 1.4M points and the rank-curve summary on the
  reference's 20k-row subsample within 1% (north star).

C4 (configs[3]): the 10^7-vertex planted graph, nn=3: 10 iterations against
the oracle (positions 1e-5, stress 1e-5, b exact).

C1 (configs[0]) and C2 (configs[1], Adadelta and Nesterov at the default
alpha): full runs against the reference's own results
(tests/golden/c1_golden.npz, c2_golden.npz from make_c1c2_golden.py).
"""

import hashlib
import os

import numpy as np
import pytest

import oracle as O
from oracle.ivhd_oracle import OracleRun

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2303_05455_b200")

M3, N3 = 1_400_000, 100


def normwise(a, b):
    den = np.abs(b).max()
    return float(np.abs(np.asarray(a) - b).max() / (den if den > 0 else 1.0))


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLDEN, "quality_c3.npz"))


@pytest.fixture(scope="module")
def c3(gold):
    from paper_2303_05455_b200 import _lib, synth

    _lib.load()
    nb, _, labels = synth.mixture_knn_graph(M3, N3, k=2, seed=0, spread=float(gold["spread"]))
    return nb, labels


def test_c3_graph_is_the_golden_input(c3, gold):
    nb, _ = c3
    assert nb.shape == (M3, 2)
    assert hashlib.sha256(np.ascontiguousarray(nb, np.int32).tobytes()).hexdigest() == str(gold["graph_sha256"])


def test_c3_ten_iterations_match_reference(c3, gold):
    nb, _ = c3
    rows = gold["rows10"]
    early = []

    def obs(it, pos, stress, params):
        early.append(np.asarray(pos)[rows].copy())

    cfg = P.EmbeddingConfig(nn=2, rn=1, c=0.1, iterations=10, seed=0)
    res = P.run_embedding(graph=P.KnnGraph(nb), config=cfg, observer=obs)
    ref_pos = gold["early_positions"]
    for k in range(10):
        assert normwise(early[k], ref_pos[k]) < 1e-5, f"iteration {k}"
    np.testing.assert_allclose(res.trace.stress, gold["trace_stress"][:10], rtol=1e-5)
    assert res.trace.step_size == list(gold["trace_b"][:10])
    # forces at the GPU's positions after 10 steps vs the oracle (float64)
    y = res.embedding.points
    conn = O.build_connections(nb[:, :2], res.state.rn_assignments)
    f = P.compute_forces(y, P.ConnectionSet(np.column_stack([conn.src, conn.dst]), conn.target, conn.rand), 0.1)
    fr = O.forces(y, conn, 0.1, threads=os.cpu_count() or 1)
    assert normwise(f, fr) < 1e-5


def test_c3_full_run_quality_matches_reference(c3, gold):
    from paper_2303_05455_b200 import metrics, synth

    nb, labels = c3
    cfg = P.EmbeddingConfig(nn=2, rn=1, c=0.1, iterations=2500, seed=0)
    res = P.run_embedding(graph=P.KnnGraph(nb), config=cfg)
    y = res.embedding.points
    # stress and every auto-adapt decision of the run
    assert res.state.stress == pytest.approx(float(gold["stress"]), rel=0.01)
    assert res.trace.step_size == list(gold["trace_b"])
    # label neighbour hit over all 1.4M points (metrics.py:254-294)
    cf_nn, cf = metrics.neighbor_hit(y, labels, nn_max=100)
    assert cf == pytest.approx(float(gold["cf"]), rel=0.01)
    for k in (1, 9, 99):
        assert cf_nn[k] == pytest.approx(float(gold["cf_nn"][k]), rel=0.01), f"cf_{k + 1}"
    # kNN preservation / neighbour gain on the reference's 20k-row subsample
    sub = gold["sub"]
    x, _ = synth.mixture_points(M3, N3, seed=0, spread=float(gold["spread"]))
    xs = x[sub].astype(np.float64)
    del x
    cur = metrics.evaluate_embedding(xs, y[sub], labels=labels[sub], nn_max=100, report_ks=(15, 100))
    got = cur.summary()
    for key, val in zip(gold["summary_keys"], gold["summary_vals"]):
        key = str(key)
        assert got[key] == pytest.approx(float(val), rel=0.01, abs=1e-3 * max(1.0, abs(float(val)))), key


def test_c4_ten_iterations_vs_oracle():
    """10^7-vertex planted graph, nn=3 rn=1 (BASELINE configs[3], one GPU)."""
    from paper_2303_05455_b200 import synth

    m = 10_000_000
    nb = synth.planted_graph(m, 3, seed=0)
    cfg = dict(nn=3, rn=1, c=0.1, iterations=10, seed=0)
    res = P.run_embedding(graph=P.KnnGraph(nb), config=P.EmbeddingConfig(**cfg))
    ref = OracleRun(nb, threads=os.cpu_count() or 1, **cfg)
    ref.run()
    assert normwise(res.embedding.points, ref.Y) < 1e-5
    np.testing.assert_allclose(res.trace.stress, ref.trace_stress, rtol=1e-5)
    assert res.trace.step_size == [float(b) for b in ref.trace_b]


def test_c1_full_run_matches_reference():
    """C1 (configs[0]): 20k x 784 mixture (spread 0.23, cf ~ 0.70), exact 2-NN
    graph from the reference's build_exact_knn, nn=2 rn=1 c=0.01, FD, 2000
    iterations — against the reference's own full run
    (tests/golden/c1_golden.npz, make_c1c2_golden.py): stress, every step
    decision, neighbour hit and the rank-curve summary over all 20k rows."""
    from paper_2303_05455_b200 import metrics, synth

    g = np.load(os.path.join(GOLDEN, "c1_golden.npz"))
    nb, labels = g["neighbors"], g["labels"].astype(np.int64)
    cfg = P.EmbeddingConfig(nn=2, rn=1, c=0.01, iterations=2000, seed=0)
    res = P.run_embedding(graph=P.KnnGraph(nb), config=cfg)
    y = res.embedding.points
    assert res.state.stress == pytest.approx(float(g["stress"]), rel=0.01)
    np.testing.assert_allclose(res.trace.stress[:10], g["trace_stress"][:10], rtol=1e-5)
    assert res.trace.step_size == list(g["trace_b"])
    cf_nn, cf = metrics.neighbor_hit(y, labels, nn_max=100)
    assert cf == pytest.approx(float(g["cf"]), rel=0.01)
    x, _ = synth.mixture_points(20000, 784, seed=0, spread=float(g["spread"]))
    got = metrics.evaluate_embedding(x.astype(np.float64), y, labels=labels, nn_max=100,
                                     report_ks=(15, 100)).summary()
    for key, val in zip(g["summary_keys"], g["summary_vals"]):
        key = str(key)
        assert got[key] == pytest.approx(float(val), rel=0.01, abs=1e-3 * max(1.0, abs(float(val)))), key


@pytest.mark.parametrize("opt", ["adadelta", "nesterov"])
def test_c2_full_run_matches_reference(opt):
    """C2 (configs[1]): the reference's mnist_like(70000, 784) exact 5-NN graph,
    nn=5 rn=1 c=0.01, 2500 iterations at the default alpha — final stress, the
    first 10 stresses and the neighbour hit against the reference's run."""
    from paper_2303_05455_b200 import metrics

    g = np.load(os.path.join(GOLDEN, "c2_golden.npz"))
    nb, labels = g["neighbors"], g["labels"].astype(np.int64)
    cfg = P.EmbeddingConfig(nn=5, rn=1, c=0.01, iterations=2500, seed=0, optimizer=opt)
    res = P.run_embedding(graph=P.KnnGraph(nb), config=cfg)
    assert res.state.stress == pytest.approx(float(g[f"{opt}_stress"]), rel=0.01)
    np.testing.assert_allclose(res.trace.stress[:10], g[f"{opt}_trace_stress"][:10], rtol=1e-5)
    assert res.trace.step_size == list(g[f"{opt}_trace_b"])
    cf_nn, cf = metrics.neighbor_hit(res.embedding.points, labels, nn_max=100)
    assert cf == pytest.approx(float(g[f"{opt}_cf"]), rel=0.01)
    assert cf_nn[9] == pytest.approx(float(g[f"{opt}_cf_nn"][9]), rel=0.01)
