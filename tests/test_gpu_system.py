"""System-level GPU tests: the NCCL sharded path, full-run quality parity
against the CPU oracle, determinism, observer/mutation flow.  Marked gpu."""

import os
import socket

import numpy as np
import pytest

from oracle.ivhd_oracle import OracleRun

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2303_05455_b200")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(m=6000, seed=0):
    from paper_2303_05455_b200 import synth

    return synth.planted_graph(m, 3, seed=seed)


def test_sharded_nccl_world1_matches_single_gpu():
    """The sharded driver (per-unit partials, standalone finalizer) against the
    fused single-GPU loop (per-thread running partials): same per-vertex math,
    so positions and step decisions agree bit for bit here; the reported
    stress differs only by the fp32 summation order of the partials."""
    import torch
    import torch.distributed as dist

    from paper_2303_05455_b200.config import resolve_optimizer
    from paper_2303_05455_b200.device import DeviceEmbedding
    from paper_2303_05455_b200.embed import init_layout, sample_random_neighbors
    from paper_2303_05455_b200.sharded import ShardedEmbedding

    nb = _problem()
    m = nb.shape[0]
    rng = np.random.default_rng(1)
    y0 = init_layout(m, 2, rng)
    rn = sample_random_neighbors(m, nb, 1, rng)
    ref = DeviceEmbedding(m, 2)
    ref.set_optimizer(resolve_optimizer("force-directed", m))
    ref.set_positions(y0)
    ref.set_graph(0, nb, rn)
    s_ref, b_ref, _, _ = ref.run(0, "l2", 0.1, 40)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        stream = torch.cuda.current_stream()
        sh = ShardedEmbedding(m, 2, 0, 1, stream=stream.cuda_stream)
        sh.set_optimizer(resolve_optimizer("force-directed", m))
        sh.set_positions(y0)
        sh.set_graph(0, nb, rn)
        s_sh, b_sh, done, div = sh.run(0, "l2", 0.1, 40)
        assert done == 40 and not div
        np.testing.assert_array_equal(sh.positions(), ref.positions())
        np.testing.assert_allclose(np.asarray(s_sh), s_ref, rtol=1e-6)
        np.testing.assert_array_equal(np.asarray(b_sh), b_ref)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("integ,iters,diverges", [
    ({"b": 0.5, "tau": 1e-6}, 30, False),   # rollback-heavy auto-adapt
    ({"b": 1e6, "auto_adapt": False}, 40, True),  # blow-up
])
def test_sharded_async_loop_rollback_and_divergence(integ, iters, diverges):
    """The asynchronous sharded loop (parity buffers, rollback refill on the
    device, status read once at the end) against the fused single-GPU loop."""
    import torch
    import torch.distributed as dist

    from paper_2303_05455_b200.config import IntegratorParams, resolve_optimizer
    from paper_2303_05455_b200.device import DeviceEmbedding
    from paper_2303_05455_b200.embed import init_layout, sample_random_neighbors
    from paper_2303_05455_b200.sharded import ShardedEmbedding

    # 6000 ids: an id-local input, so the sharded and the fused loop use the
    # same (windowed) vertex order and agree bit for bit even while blowing up
    nb = _problem(6000)
    m = nb.shape[0]
    rng = np.random.default_rng(2)
    y0 = init_layout(m, 2, rng)
    rn = sample_random_neighbors(m, nb, 1, rng)
    opt = resolve_optimizer("force-directed", m, IntegratorParams(**integ))
    ref = DeviceEmbedding(m, 2)
    ref.set_optimizer(opt)
    ref.set_positions(y0)
    ref.set_graph(0, nb, rn)
    s_ref, b_ref, d_ref, div_ref = ref.run(0, "l2", 0.1, iters)
    assert div_ref == diverges
    if not diverges:
        assert (b_ref[1:] != b_ref[:-1]).sum() >= 3

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        stream = torch.cuda.current_stream()
        sh = ShardedEmbedding(m, 2, 0, 1, stream=stream.cuda_stream)
        sh.set_optimizer(opt)
        sh.set_positions(y0)
        sh.set_graph(0, nb, rn)
        s_sh, b_sh, done, div = sh.run(0, "l2", 0.1, iters)
        assert div == diverges and done == d_ref
        np.testing.assert_array_equal(np.asarray(b_sh), b_ref)
        np.testing.assert_allclose(np.asarray(s_sh)[np.isfinite(s_ref)], s_ref[np.isfinite(s_ref)], rtol=1e-5)
        np.testing.assert_array_equal(sh.positions(), ref.positions())
    finally:
        dist.destroy_process_group()


def _knn_preservation(Y, nb, k=2):
    """Fraction of graph neighbours among each point's k nearest in 2-D."""
    from scipy.spatial import cKDTree

    _, idx = cKDTree(Y).query(Y, k=k + 1)
    hits = [len(set(idx[i, 1:]) & set(nb[i, :k])) for i in range(len(Y))]
    return float(np.mean(hits)) / k


def _neighbor_hit(Y, labels, k=10):
    from scipy.spatial import cKDTree

    _, idx = cKDTree(Y).query(Y, k=k + 1)
    return float((labels[idx[:, 1:]] == labels[:, None]).mean())


def test_full_run_quality_matches_oracle_within_1pct():
    """North star: after a full run the stress and the kNN-preservation /
    neighbour-hit quality agree with the CPU reference within 1%."""
    import torch

    from paper_2303_05455_b200 import synth

    m = 4000
    nb, _, labels = synth.mixture_knn_graph(m, 20, k=2, clusters=6, seed=3)
    cfg = dict(nn=2, rn=1, c=0.1, iterations=600, seed=0)
    res = P.run_embedding(graph=P.KnnGraph(nb), config=P.EmbeddingConfig(**cfg))
    ref = OracleRun(nb, **cfg)
    ref.run()
    assert res.state.stress == pytest.approx(ref.trace_stress[-1], rel=1e-2)
    q_gpu, q_ref = _knn_preservation(res.embedding.points, nb), _knn_preservation(ref.Y, nb)
    h_gpu, h_ref = _neighbor_hit(res.embedding.points, labels), _neighbor_hit(ref.Y, labels)
    assert abs(q_gpu - q_ref) <= 0.01 * max(q_ref, 1e-9) + 1e-3
    assert abs(h_gpu - h_ref) <= 0.01 * h_ref
    torch.cuda.synchronize()


def test_observer_stop_and_mutations_on_device():
    nb = _problem(2000)
    seen = []

    def obs(it, pos, stress, params):
        seen.append((it, params["b"], params["c"]))
        if it == 3:
            return {"c": 0.05, "b": 0.004}
        if it == 9:
            return {"stop": True}

    res = P.run_embedding(graph=P.KnnGraph(nb), config=P.EmbeddingConfig(nn=3, rn=1, iterations=100),
                          observer=obs)
    assert len(res.trace.iterations) == 10
    assert (3, "c", 0.05) in res.mutations and (3, "b", 0.004) in res.mutations
    assert seen[4][2] == 0.05
    # iteration 4 stepped with b = 0.004 (then possibly adapted by gamma1/gamma2)
    assert any(seen[4][1] == pytest.approx(0.004 * g) for g in (1.0, 1.1, 0.9))


def test_optimizer_swap_mid_run_keeps_positions():
    nb = _problem(2000)

    def obs(it, pos, stress, params):
        if it == 4:
            return {"optimizer": "nesterov"}

    res = P.run_embedding(graph=P.KnnGraph(nb), config=P.EmbeddingConfig(nn=3, rn=1, iterations=20),
                          observer=obs)
    assert (4, "optimizer", "nesterov") in res.mutations
    assert np.isfinite(res.embedding.points).all()


def test_large_graph_runs_and_is_deterministic():
    nb = _problem(300_000)
    cfg = P.EmbeddingConfig(nn=3, rn=1, c=0.1, iterations=150, seed=2)
    a = P.run_embedding(graph=P.KnnGraph(nb), config=cfg)
    b = P.run_embedding(graph=P.KnnGraph(nb), config=cfg)
    np.testing.assert_array_equal(a.embedding.points, b.embedding.points)
    assert a.trace.stress == b.trace.stress
    assert a.trace.stress[-1] < a.trace.stress[0]


@pytest.mark.gpu
def test_observer_positions_are_lazy_and_pinned_when_kept():
    """Steering fast path: positions reach the host only when the observer
    reads them; a kept reference still holds its own iteration's values."""
    import time

    from paper_2303_05455_b200 import EmbeddingConfig, KnnGraph, run_embedding, synth

    nb = synth.planted_graph(50_000, 2, seed=1)
    cfg = EmbeddingConfig(nn=2, rn=1, c=0.1, iterations=60, seed=3)
    eager = {}
    run_embedding(graph=KnnGraph(nb), config=cfg,
                  observer=lambda it, p, e, prm: eager.__setitem__(it, np.array(p)))
    kept, framed = {}, {}

    def obs(it, p, e, prm):
        kept[it] = p  # retained proxy: must be pinned to iteration `it`
        if it % 10 == 0:
            framed[it] = np.asarray(p).copy()

    run_embedding(graph=KnnGraph(nb), config=cfg, observer=obs)
    for it in framed:
        np.testing.assert_array_equal(framed[it], eager[it])
    for it in (0, 7, 31, 59):
        np.testing.assert_array_equal(np.asarray(kept[it]), eager[it])
    # frame every 50 iterations: the per-iteration device round trip without a
    # full position copy (recorded, not asserted: timing is informative only)
    def framer(it, p, e, prm):
        if it % 50 == 0:
            np.asarray(p).sum()

    t0 = time.perf_counter()
    run_embedding(graph=KnnGraph(nb), config=EmbeddingConfig(nn=2, rn=1, c=0.1, iterations=300, seed=3),
                  observer=framer)
    print(f"observer fast path: {(time.perf_counter() - t0) / 300 * 1e6:.0f} us/iteration")


@pytest.mark.gpu
def test_run_embedding_builds_graph_from_dataset():
    """engine.py:170-176 / 194-199: without a graph, run_embedding builds the
    exact kNN graph (and the 4*nn helper for the RNN phase) from the dataset —
    here on the GPU — and the run equals one given that graph explicitly."""
    from types import SimpleNamespace

    from paper_2303_05455_b200 import EmbeddingConfig, run_embedding
    from paper_2303_05455_b200.knng import build_exact_knn

    rng = np.random.default_rng(8)
    x = rng.standard_normal((3000, 20)) + 3.0 * rng.standard_normal((6, 20))[rng.integers(0, 6, 3000)]
    ds = SimpleNamespace(data=x, labels=None)
    cfg = EmbeddingConfig(nn=3, rn=1, c=0.1, iterations=40, seed=5)
    a = run_embedding(dataset=ds, config=cfg)
    b = run_embedding(graph=build_exact_knn(x, 3), config=cfg)
    np.testing.assert_array_equal(a.embedding.points, b.embedding.points)
    cfg2 = EmbeddingConfig(nn=3, rn=1, c=0.1, iterations=40, seed=5, rnn_final_steps=10)
    c = run_embedding(dataset=ds, config=cfg2)
    d = run_embedding(graph=build_exact_knn(x, 3), helper_graph=build_exact_knn(x, 12), dataset=ds, config=cfg2)
    np.testing.assert_array_equal(c.embedding.points, d.embedding.points)


def test_c2_fixture_quality_matches_reference_within_1pct():
    """North star acceptance on SURVEY §8(d)'s discriminating C2 fixture
    (mnist_like 70k -> PCA 100 -> exact 2-NN graph, nn=2 rn=1 c=0.01, FD,
    2500 iterations; tests/golden/make_quality_golden.py): final stress,
    neighbour hit (cf, cf_2, cf_10 over all 70k points) and the rank-curve
    metrics on a fixed 2000-row subsample (AUC R_NX, AUC G_NN, trust /
    continuity at 15 and 100) agree with the reference's run within 1%."""
    import os

    from paper_2303_05455_b200 import metrics
    from tests.golden.make_quality_golden import OUT, subsample

    g = np.load(OUT)
    nb, labels = g["neighbors"], g["labels"].astype(np.int64)
    cfg = P.EmbeddingConfig(nn=2, rn=1, c=0.01, iterations=2500, seed=0)
    res = P.run_embedding(graph=P.KnnGraph(nb), config=cfg)
    y = res.embedding.points
    assert res.state.stress == pytest.approx(float(g["stress"]), rel=1e-2)
    cf_nn, cf = metrics.neighbor_hit(y, labels, nn_max=100)
    ref_nn = g["cf_nn"]
    for got, want in ((cf, ref_nn.mean()), (cf_nn[1], ref_nn[1]), (cf_nn[9], ref_nn[9])):
        assert got == pytest.approx(float(want), rel=1e-2)
    sub = subsample()
    cur = metrics.evaluate_embedding(g["x_sub"], y[sub], labels=labels[sub], report_ks=(15, 100))
    print(os.linesep, cur.summary(), float(g["auc_rnx"]), float(g["auc_gnn"]), g["trust"], g["continuity"])
    assert cur.auc_rnx == pytest.approx(float(g["auc_rnx"]), rel=1e-2)
    assert cur.auc_gnn == pytest.approx(float(g["auc_gnn"]), rel=1e-2)
    np.testing.assert_allclose([cur.trust[15], cur.trust[100]], g["trust"], rtol=1e-2)
    np.testing.assert_allclose([cur.continuity[15], cur.continuity[100]], g["continuity"], rtol=1e-2)


def test_result_arrays_in_recycled_pinned_buffers():
    """run_embedding's result arrays come from the pinned pool: independent
    buffers (the embedding is its own copy, engine.py:413), recycled once the
    arrays die, values equal across runs."""
    import gc

    from paper_2303_05455_b200 import _lib, synth

    nb = synth.planted_graph(200_000, 2, seed=1)
    cfg = P.EmbeddingConfig(nn=2, rn=1, c=0.1, iterations=20, seed=0)
    r1 = P.run_embedding(graph=P.KnnGraph(nb), config=cfg)
    pts, pos, dl = r1.embedding.points, r1.state.positions, r1.state.deltas
    assert pts.ctypes.data != pos.ctypes.data and pos.ctypes.data != dl.ctypes.data
    np.testing.assert_array_equal(pts, pos)
    keep = pts.copy()
    pos[0, 0] += 1.0
    assert pts[0, 0] == keep[0, 0]
    addrs = {pts.ctypes.data, pos.ctypes.data, dl.ctypes.data}
    del r1, pts, pos, dl
    gc.collect()
    r2 = P.run_embedding(graph=P.KnnGraph(nb), config=cfg)
    assert {r2.embedding.points.ctypes.data, r2.state.positions.ctypes.data, r2.state.deltas.ctypes.data} == addrs
    np.testing.assert_array_equal(r2.embedding.points, keep)
    assert _lib.pinned._outstanding == 3 * 200_000 * 2 * 8


def test_pinned_pool_cap_releases_pooled_buffers():
    import gc

    from paper_2303_05455_b200._lib import PinnedPool

    mib = 1 << 20
    p = PinnedPool(cap_bytes=5 * mib)
    a = p.empty((mib // 16, 2))  # 1 MiB... (8 bytes x 2 x mib/16 = 1 MiB)
    b = p.empty((mib // 8, 2))   # 2 MiB
    assert p._outstanding == 3 * mib
    c = p.empty((mib // 8, 2))   # 2 MiB more would reach 5 MiB: still fits
    assert p._outstanding == 5 * mib
    d = p.empty((mib // 16, 2))  # over the cap: plain numpy
    assert p._outstanding == 5 * mib and d.shape == (mib // 16, 2)
    del a, b
    gc.collect()
    assert p._outstanding == 2 * mib and p._pooled == 3 * mib
    e = p.empty((3 * mib // 16, 2))  # 3 MiB: pooled 1 + 2 MiB buffers are released for it
    assert p._outstanding == 5 * mib and p._pooled == 0
    e[...] = 1.0
    c[...] = 2.0
    assert float(e.sum()) == e.size and float(c.sum()) == 2 * c.size


@pytest.mark.parametrize("phased", [False, True])
def test_run_embedding_distributed_world1_matches_run_embedding(phased):
    """The public multi-GPU entry point (sharded.run_embedding_distributed) on
    a one-rank NCCL group: same RunResult contract and trajectory as
    run_embedding on a hub-heavy mixture kNN graph (snake-dealt rank groups:
    a different vertex order, so equal to fp32 summation order).  phased: rn
    resampling, the RNN-filtered phase (weighted connection set) and the L1
    phase through the sharded (peer) kernels."""
    import torch
    import torch.distributed as dist

    from paper_2303_05455_b200 import synth
    from paper_2303_05455_b200.sharded import run_embedding_distributed

    nb, _, _ = synth.mixture_knn_graph(30000, 50, k=12, seed=3, spread=0.5)  # k = 4 nn: its own RNN helper
    extra = dict(rn_resample_period=7, rnn_final_steps=10, l1_final_steps=8) if phased else {}
    cfg = P.EmbeddingConfig(nn=3, rn=1, c=0.1, iterations=50, seed=5, **extra)
    a = P.run_embedding(graph=P.KnnGraph(nb), config=cfg)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        b = run_embedding_distributed(graph=P.KnnGraph(nb), config=cfg)
    finally:
        dist.destroy_process_group()
    assert b.state.iteration == 50 and len(b.trace.stress) == 50
    assert np.abs(b.embedding.points - a.embedding.points).max() / np.abs(a.embedding.points).max() < 1e-5
    np.testing.assert_allclose(b.trace.stress, a.trace.stress, rtol=1e-5)
    assert b.trace.step_size == a.trace.step_size
    np.testing.assert_array_equal(b.state.rn_assignments, a.state.rn_assignments)


@pytest.mark.parametrize("dim,opt", [(2, "force-directed"), (2, "nesterov"), (3, "force-directed"),
                                     (3, "nesterov")])
def test_gather_floor_is_below_the_step_time(dim, opt):
    """ivhd_gather_floor: the gather-only pass over the CSR takes less device
    time than a full iteration on the same graph (positive, finite), for every
    position record width (2-D / 3-D, with Nesterov's look-ahead: 2, 4, 8 floats)."""
    import time

    from paper_2303_05455_b200.config import resolve_optimizer
    from paper_2303_05455_b200.device import DeviceEmbedding
    from paper_2303_05455_b200.embed import init_layout, sample_random_neighbors

    nb = _problem(200_000)
    m = nb.shape[0]
    rng = np.random.default_rng(0)
    dev = DeviceEmbedding(m, dim)
    dev.set_optimizer(resolve_optimizer(opt, m))
    dev.set_positions(init_layout(m, dim, rng))
    dev.set_graph(0, nb[:, :3], sample_random_neighbors(m, nb[:, :3], 1, rng))
    g = dev.gather_floor(0, reps=5)
    dev.run(0, "l2", 0.1, 50)
    dev.synchronize()
    t0 = time.perf_counter()
    dev.run(0, "l2", 0.1, 200)
    dev.synchronize()
    per_iter = (time.perf_counter() - t0) / 200 * 1e6
    dev.close()
    assert 0.0 < g < per_iter
    fresh = DeviceEmbedding(m, dim)
    with pytest.raises(P.DeviceError, match="not set"):
        fresh.gather_floor(0)  # no connection set yet
    with pytest.raises(P.InvalidArgumentError):
        fresh.gather_floor(2)
    fresh.close()
