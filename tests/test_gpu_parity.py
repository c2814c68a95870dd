"""Parity of the CUDA path against the reference (golden fixtures made by the
reference itself) and the CPU oracle.  Needs a B200: marked gpu.

Tolerances (north star): per-iteration forces and positions within 1e-5
normwise relative (max|x - ref| / max|ref|, the reference's own definition,
test_forces.py:135) for 10 steps; after a full run, stress and quality
metrics within 1%.
"""

import json
import os

import numpy as np
import pytest

import oracle as O
from oracle.ivhd_oracle import OracleRun

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2303_05455_b200")


def normwise(a, b):
    den = np.abs(b).max()
    return float(np.abs(np.asarray(a) - b).max() / (den if den > 0 else 1.0))


def load(name):
    return np.load(os.path.join(GOLDEN, name))


META = json.load(open(os.path.join(GOLDEN, "meta.json")))
FC = load("force_cases.npz")
N_CASES = int(FC["n_cases"])
BLOB = load("blob_graph.npz")


@pytest.fixture(scope="module", autouse=True)
def _lib_loaded():
    from paper_2303_05455_b200 import _lib

    _lib.load()  # fail loudly if the CUDA library is missing


# ----------------------------------------------------------- operator level


@pytest.mark.parametrize("k", range(N_CASES))
def test_forces_match_reference_golden(k):
    p = f"c{k}_"
    sc = FC[p + "scale"]
    conn = P.ConnectionSet(FC[p + "edges"], FC[p + "targets"], FC[p + "is_random"],
                           None if sc.size == 0 else sc)
    Y, c, norm = FC[p + "Y"], float(FC[p + "c"]), str(FC[p + "norm"])
    f, e = P.compute_forces(Y, conn, c, norm, with_stress=True)
    assert normwise(f, FC[p + "force"]) < 1e-5
    assert e == pytest.approx(float(FC[p + "stress_with"]), rel=1e-5)
    assert P.stress(Y, conn, c, norm) == pytest.approx(float(FC[p + "stress"]), rel=1e-5)


def test_hand_values():
    """test_forces.py:98-125 hand values through the CUDA operator."""
    def pair(t, rnd):
        return P.ConnectionSet(np.array([[0, 1]]), np.array([t]), np.array([rnd]))

    f = P.compute_forces(np.zeros((2, 2)), pair(0.0, False), c=0.5)
    np.testing.assert_array_equal(f, 0.0)
    f = P.compute_forces(np.array([[3.0, 4.0], [0.0, 0.0]]), pair(0.0, False), c=0.5)
    np.testing.assert_allclose(f[0], [-3.0, -4.0], rtol=1e-6)
    np.testing.assert_allclose(f[1], [3.0, 4.0], rtol=1e-6)
    f = P.compute_forces(np.array([[0.0, 0.0], [1.0, 0.0]]), pair(1.0, True), c=0.1)
    np.testing.assert_allclose(f, 0.0, atol=1e-7)
    f = P.compute_forces(np.array([[0.0, 0.0], [0.5, 0.0]]), pair(1.0, True), c=0.1)
    assert f[0, 0] < 0 < f[1, 0]
    # degenerate random pair: the reference's default_rng(0) direction, magnitude w*t
    f = P.compute_forces(np.zeros((2, 2)), pair(1.0, True), c=0.1)
    u = np.random.default_rng(0).standard_normal((1, 2))
    u /= np.linalg.norm(u)
    np.testing.assert_allclose(f[0], 0.1 * u[0], rtol=1e-6)
    np.testing.assert_allclose(f[1], -0.1 * u[0], rtol=1e-6)
    assert P.stress(np.zeros((2, 2)), pair(1.0, True), c=0.1) == pytest.approx(0.1, rel=1e-6)
    assert P.stress(np.array([[0.0, 0.0], [2.0, 0.0]]), pair(0.0, False), c=0.5) == pytest.approx(4.0)


def test_unknown_norm():
    conn = P.ConnectionSet(np.array([[0, 1]]), np.array([0.0]), np.array([False]))
    with pytest.raises(P.InvalidArgumentError):
        P.stress(np.zeros((2, 2)), conn, 0.1, "l3")


def test_out_of_range_ids_raise():
    conn = P.ConnectionSet(np.array([[0, 5]]), np.array([0.0]), np.array([False]))
    with pytest.raises(P.InvalidArgumentError):
        P.compute_forces(np.zeros((2, 2)), conn, 0.1)


# ----------------------------------------------------- 10-step loop replays


REPLAYS = sorted(k for k in META if k.startswith("replay_"))


@pytest.mark.parametrize("name", REPLAYS)
def test_ten_steps_match_reference(name):
    meta = META[name]
    g = load(name + ".npz")
    graph = P.KnnGraph(BLOB["neighbors"])
    cfg = P.EmbeddingConfig(nn=meta["nn"], rn=meta["rn"], c=meta["c"], iterations=meta["steps"],
                            seed=meta["seed"], optimizer=meta["optimizer"],
                            target_dim=meta["target_dim"])
    seen = []
    res = P.run_embedding(graph=graph, config=cfg,
                          observer=lambda it, pos, s, prm: seen.append((pos.copy(), s, prm["b"])))
    assert len(seen) == meta["steps"]
    np.testing.assert_array_equal(res.state.rn_assignments, g["rn"])
    for s, (pos, e, b) in enumerate(seen):
        assert normwise(pos, g["positions"][s]) < 1e-5, f"step {s}"
        assert e == pytest.approx(float(g["stress"][s]), rel=1e-5)
        assert b == pytest.approx(float(g["b"][s]), rel=1e-6)
    # forces at the reference's evaluation points of every step
    conn = P.ConnectionSet(
        np.column_stack([np.repeat(np.arange(graph.M), 4),
                         np.column_stack([graph.neighbors[:, :3], g["rn"]]).ravel()]),
        np.tile([0.0, 0.0, 0.0, 1.0], graph.M), np.tile([False, False, False, True], graph.M))
    prev = g["Y0"]
    before = g["Y0"]
    for s in range(meta["steps"]):
        ev = before
        if meta["optimizer"] == "nesterov":
            ev = before + 0.9 * (before - prev)
        f = P.compute_forces(ev, conn, meta["c"])
        assert normwise(f, g["force"][s]) < 1e-5, f"forces step {s}"
        prev, before = before, g["positions"][s]


# -------------------------------------------------------------- full runs


RUNS = sorted(k[4:] for k in META if k.startswith("run_") and k != "run_diverge")


@pytest.mark.parametrize("name", RUNS)
def test_full_run_matches_reference(name):
    kw = dict(META["run_" + name])
    g = load(f"run_{name}.npz")
    graph = P.KnnGraph(BLOB["neighbors"], BLOB["distances"])
    ds = None
    if kw.get("distance_mode") == "euclidean":
        class _D:
            data = BLOB["data"]
            labels = None
        ds = _D()
    res = P.run_embedding(graph=graph, config=P.EmbeddingConfig(**kw), dataset=ds)
    np.testing.assert_array_equal(res.state.rn_assignments, g["rn"])
    assert res.state.iteration == int(g["iteration"])
    if kw["iterations"] == 0:
        np.testing.assert_array_equal(res.embedding.points, g["points"])
        assert res.state.stress == pytest.approx(float(g["final_stress"]), rel=1e-5)
        return
    # the step-size trace (auto-adapt decisions) is reproduced exactly
    np.testing.assert_allclose(res.trace.step_size, g["b"], rtol=1e-6)
    assert res.trace.stress[-1] == pytest.approx(float(g["stress"][-1]), rel=1e-2)
    assert res.state.stress == pytest.approx(float(g["final_stress"]), rel=1e-2)
    assert normwise(res.embedding.points, g["points"]) < 1e-2


def test_divergence_carries_last_finite_state():
    kw = META["run_diverge"]
    g = load("run_diverge.npz")
    cfg = P.EmbeddingConfig(**{**kw, "integrator": P.IntegratorParams(**kw["integrator"])})
    with pytest.raises(P.NumericalDivergenceError) as err:
        P.run_embedding(graph=P.KnnGraph(BLOB["neighbors"]), config=cfg)
    # float32 overflows (3.4e38) long before float64 (1.8e308): with b=1e6 the
    # blow-up is detected at an earlier iteration than in the reference, but
    # the contract is the same — raise with the last finite pre-step state.
    assert 0 <= err.value.iteration <= int(g["iteration"])
    st = err.value.state
    assert np.isfinite(st.positions).all()
    assert st.iteration == err.value.iteration


def test_repeat_runs_bit_identical():
    cfg = P.EmbeddingConfig(nn=3, rn=1, c=0.1, iterations=200, seed=3)
    graph = P.KnnGraph(BLOB["neighbors"])
    a = P.run_embedding(graph=graph, config=cfg)
    b = P.run_embedding(graph=graph, config=cfg)
    np.testing.assert_array_equal(a.embedding.points, b.embedding.points)
    assert a.trace.stress == b.trace.stress


# ------------------------------------------------ larger graphs vs oracle


def planted_graph(m, k, seed=0, clusters=10, span=63):
    """SURVEY appendix planted kNN-shaped graph (locality, no hubs)."""
    rng = np.random.default_rng(seed)
    size = m // clusters
    ids = np.arange(m)
    base = np.minimum(ids // size, clusters - 1) * size
    csize = np.where(ids // size >= clusters - 1, m - (clusters - 1) * size, size)
    off = rng.integers(1, span + 1, size=(m, k))
    return ((ids[:, None] - base[:, None] + off) % csize[:, None] + base[:, None]).astype(np.int32)


@pytest.mark.parametrize("m,nn,opt", [(20000, 2, "force-directed"), (70000, 5, "adadelta"),
                                      (70000, 5, "nesterov"), (50000, 3, "adam"),
                                      (30000, 3, "momentum"), (30000, 2, "sgd")])
def test_ten_steps_vs_oracle_at_scale(m, nn, opt):
    nb = planted_graph(m, nn)
    cfg = dict(nn=nn, rn=1, c=0.01, iterations=10, seed=0, optimizer=opt)
    res = P.run_embedding(graph=P.KnnGraph(nb), config=P.EmbeddingConfig(**cfg))
    ref = OracleRun(nb, **cfg)
    ref.run()
    # Adam runs the float64 kernel (ivhd_step_f64.cuh): its division by the
    # running RMS gradient would amplify fp32 rounding of nearly cancelled
    # components; every optimizer is held to the north star's 1e-5
    assert normwise(res.embedding.points, ref.Y) < 1e-5
    np.testing.assert_allclose(res.trace.stress, ref.trace_stress, rtol=1e-5)
    # forces at the oracle's final positions: 1e-5 for every optimizer
    f = P.compute_forces(ref.Y, P.ConnectionSet(np.column_stack([ref.full.src, ref.full.dst]),
                                                ref.full.target, ref.full.rand), 0.01)
    fr = O.forces(ref.Y, ref.full, 0.01)
    assert normwise(f, fr) < 1e-5


def test_locality_ordered_graph_repeat_runs_bit_identical():
    # a planted graph has >= 50% id-local connections, so the library picks the
    # windowed degree order and the in-order schedule (ivhd_capi.cu fix_permutation)
    nb = planted_graph(60000, 2)
    cfg = P.EmbeddingConfig(nn=2, rn=1, c=0.1, iterations=100, seed=1)
    a = P.run_embedding(graph=P.KnnGraph(nb), config=cfg)
    b = P.run_embedding(graph=P.KnnGraph(nb), config=cfg)
    np.testing.assert_array_equal(a.embedding.points, b.embedding.points)
    assert a.trace.stress == b.trace.stress
    ref = OracleRun(nb, nn=2, rn=1, c=0.1, iterations=10, seed=1)
    ref.run()
    c = P.run_embedding(graph=P.KnnGraph(nb), config=P.EmbeddingConfig(nn=2, rn=1, c=0.1, iterations=10, seed=1))
    assert normwise(c.embedding.points, ref.Y) < 1e-5


@pytest.mark.parametrize("m,dim", [(20000, 3), (40000, 2)])
def test_adam_float64_path_ten_steps(m, dim):
    """Adam (optim.py:178-205) runs the float64 kernel: positions and the
    stress trace agree with the oracle at the north star's 1e-5 per step, in
    2-D and 3-D (3-D state is 8 doubles per vertex)."""
    nb = planted_graph(m, 3, seed=1)
    cfg = dict(nn=3, rn=1, c=0.05, iterations=10, seed=2, optimizer="adam", target_dim=dim)
    res = P.run_embedding(graph=P.KnnGraph(nb), config=P.EmbeddingConfig(**cfg))
    ref = OracleRun(nb, **cfg)
    for k in range(10):
        ref.step()
    assert normwise(res.embedding.points, ref.Y) < 1e-5
    np.testing.assert_allclose(res.trace.stress, ref.trace_stress, rtol=1e-5)


def test_switch_force_directed_to_adam_mid_run():
    """An observer switches the optimizer to Adam after 5 iterations
    (engine.py:417-448): the fp32 positions are re-packed into the fp64
    layout and Adam starts from fresh state.  The force-directed prefix is
    held to 1e-5; the Adam phase is compared with an oracle restarted from
    the GPU's own positions at the switch (Adam would otherwise amplify the
    prefix's fp32 rounding, see test_adam_float64_path_ten_steps)."""
    from oracle.ivhd_oracle import make_state

    nb = planted_graph(30000, 2, seed=3)
    cfg = dict(nn=2, rn=1, c=0.1, iterations=10, seed=4)
    seen = {}

    def obs(it, pos, stress, params):
        if it == 4:
            seen["y"] = np.array(pos)
            return {"optimizer": "adam"}
        return None

    res = P.run_embedding(graph=P.KnnGraph(nb), config=P.EmbeddingConfig(**cfg), observer=obs)
    ref = OracleRun(nb, **cfg)
    for _ in range(5):
        ref.step()
    assert normwise(seen["y"], ref.Y) < 1e-5
    ref.Y = seen["y"].copy()
    ref.opt = make_state("adam", ref.m, 2)
    for _ in range(5):
        ref.step()
    assert normwise(res.embedding.points, ref.Y) < 1e-5
    np.testing.assert_allclose(res.trace.stress, ref.trace_stress, rtol=1e-5)


# ---------------------------------------- degenerate random pairs (a8)

DEG = load("degenerate_cases.npz")


@pytest.mark.parametrize("k", range(int(DEG["n_cases"])))
def test_degenerate_pairs_match_reference_golden(k):
    """forces.py:158-174 through the CUDA operator: the kernel reports the
    zero-distance random pairs, the host draws their directions from `rng`
    (default_rng(0) when None) in connection order, the kernel applies them."""
    p = f"d{k}_"
    sc = DEG[p + "scale"]
    conn = P.ConnectionSet(DEG[p + "edges"], DEG[p + "targets"], DEG[p + "is_random"],
                           None if sc.size == 0 else sc)
    seed = int(DEG[p + "seed"])
    gen = None if seed < 0 else np.random.default_rng(seed)
    f, e = P.compute_forces(DEG[p + "Y"], conn, float(DEG[p + "c"]), rng=gen, with_stress=True)
    assert normwise(f, DEG[p + "force"]) < 1e-5
    assert e == pytest.approx(float(DEG[p + "stress"]), rel=1e-5)
    if gen is not None:  # the draw consumed the caller's generator like the reference's
        ref = np.random.default_rng(seed)
        n_bad = 0
        y = DEG[p + "Y"]
        ed = DEG[p + "edges"]
        t = DEG[p + "targets"]
        n_bad = int(((np.abs(y[ed[:, 0]] - y[ed[:, 1]]).sum(1) == 0) & (t != 0)).sum())
        ref.standard_normal((n_bad, y.shape[1]))
        assert gen.bit_generator.state == ref.bit_generator.state


@pytest.mark.parametrize("opt", ["force-directed", "nesterov", "adam"])
def test_loop_pauses_for_degenerate_pairs_and_follows_the_oracle(opt):
    """The loop meets random pairs at zero distance (several rn partners
    placed on their source vertex): the iteration pauses on the device
    (nothing committed, state double buffer not advanced), the host draws the
    directions from the run's generator in connection order, the iteration is
    re-run — positions, stress and the generator state then follow the
    oracle (the reference's draw) step by step."""
    from paper_2303_05455_b200 import degenerate
    from paper_2303_05455_b200.config import resolve_optimizer
    from paper_2303_05455_b200.device import DeviceEmbedding

    nb = planted_graph(5000, 2, seed=4)
    orc = OracleRun(nb, nn=2, rn=1, c=0.1, iterations=6, seed=9, optimizer=opt)
    y0 = orc.Y.copy()
    src = np.arange(0, 5000, 97)
    y0[orc.rn_assign[src, 0]] = y0[src]  # coincident random pairs
    orc.Y = y0.copy()
    gen = np.random.Generator(np.random.PCG64())
    gen.bit_generator.state = orc.rng.bit_generator.state
    conn = orc.full
    dev = DeviceEmbedding(5000, 2)
    dev.set_optimizer(resolve_optimizer(opt, 5000))
    dev.set_positions(y0)
    dev.set_graph(0, nb, orc.rn_assign)
    calls = []

    def resolver(slot, rows, entries):
        calls.append(len(rows))
        return degenerate.table(rows, entries, conn.src, conn.dst, conn.weights(0.1) * conn.target, gen, 2)

    dev.degenerate_resolver = resolver
    st, bb, done, div = dev.run(0, "l2", 0.1, 6)
    assert done == 6 and not div and calls and calls[0] >= 2 * len(src) - 4
    orc.run(6)
    assert normwise(dev.positions(), orc.Y) < 1e-5
    np.testing.assert_allclose(st, orc.trace_stress, rtol=1e-5)
    assert gen.bit_generator.state == orc.rng.bit_generator.state
    dev.close()
