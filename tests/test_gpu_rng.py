"""Device draws of the run's initial layout and random partners against
numpy itself (engine.py:124-146 use one numpy PCG64 Generator): values and
the Generator state afterwards must be bit-identical."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2303_05455_b200")

from paper_2303_05455_b200.device import DeviceEmbedding  # noqa: E402
from paper_2303_05455_b200.embed import init_layout, sample_random_neighbors  # noqa: E402


def _gen(seed, pre):
    g = np.random.default_rng(seed)
    if pre:  # leave a buffered 32-bit half (has_uint32 = 1) or an advanced stream
        g.integers(0, 1000, size=pre)
    return g


@pytest.mark.parametrize("m,dim,seed,pre", [(1, 2, 0, 0), (1000, 2, 1, 0), (4097, 3, 2, 1),
                                           (250_000, 2, 3, 3), (1_000_003, 2, 7, 0)])
def test_init_positions_match_numpy_uniform(m, dim, seed, pre):
    ga, gb = _gen(seed, pre), _gen(seed, pre)
    dev = DeviceEmbedding(m, dim)
    dev.init_positions(ga)
    ref = init_layout(m, dim, gb)
    np.testing.assert_array_equal(dev.positions(), ref.astype(np.float32).astype(np.float64))
    assert ga.bit_generator.state == gb.bit_generator.state
    dev.close()


@pytest.mark.parametrize("m,ncols,rn,seed,pre", [
    (12, 5, 3, 0, 0),          # collisions everywhere: many re-draw rounds
    (50, 5, 1, 1, 1),          # buffered half at the start
    (1000, 2, 1, 2, 0),
    (1000, 3, 0, 3, 0),        # no random partners
    (65_537, 4, 2, 4, 5),
    (1_400_000, 2, 1, 0, 0),   # C3 shape: hundreds of Lemire rejections
    (3_000_017, 2, 3, 9, 1),
])
def test_sampled_partners_match_numpy(m, ncols, rn, seed, pre):
    rng = np.random.default_rng(100 + seed)
    nn = rng.integers(0, m, size=(m, ncols)).astype(np.int32)
    ga, gb = _gen(seed, pre), _gen(seed, pre)
    dev = DeviceEmbedding(m, 2)
    dev.init_positions(ga)
    picks = dev.set_graph_sampled(0, nn, rn, ga)
    init_layout(m, 2, gb)
    ref = sample_random_neighbors(m, nn, rn, gb)
    np.testing.assert_array_equal(picks, ref)
    assert ga.bit_generator.state == gb.bit_generator.state
    # the stream continues identically (the next resample)
    if m < 100_000:
        again = dev.set_graph_sampled(0, nn, rn, ga)
        np.testing.assert_array_equal(again, sample_random_neighbors(m, nn, rn, gb))
        assert ga.bit_generator.state == gb.bit_generator.state
    dev.close()


def test_sampled_graph_equals_host_drawn_graph():
    """The CSR built from device picks is the one built from host picks: a
    run from each is bit-identical."""
    from paper_2303_05455_b200 import synth
    from paper_2303_05455_b200.config import resolve_optimizer

    nb = synth.planted_graph(20_000, 3, seed=5)
    m = nb.shape[0]
    out = []
    for device_draws in (True, False):
        g = np.random.default_rng(11)
        dev = DeviceEmbedding(m, 2)
        dev.set_optimizer(resolve_optimizer("force-directed", m))
        if device_draws:
            dev.init_positions(g)
            dev.set_graph_sampled(0, nb, 1, g)
        else:
            dev.set_positions(init_layout(m, 2, g))
            dev.set_graph(0, nb, sample_random_neighbors(m, nb, 1, g))
        s, b, _, _ = dev.run(0, "l2", 0.1, 50)
        out.append((dev.positions(), s, b))
        dev.close()
    np.testing.assert_array_equal(out[0][0], out[1][0])
    np.testing.assert_array_equal(out[0][1], out[1][1])


def test_run_embedding_draws_match_reference_stream():
    """run_embedding's rn_assignments and resampled partners follow the
    reference's stream (rn_resample_period re-draws from the same Generator)."""
    from paper_2303_05455_b200 import synth

    nb = synth.planted_graph(5000, 3, seed=1)
    cfg = P.EmbeddingConfig(nn=3, rn=1, iterations=30, seed=4, rn_resample_period=10)
    res = P.run_embedding(graph=P.KnnGraph(nb), config=cfg)
    g = np.random.default_rng(4)
    init_layout(5000, 2, g)
    rn = None
    for _ in range(3):  # initial draw + resamples at 10 and 20
        rn = sample_random_neighbors(5000, nb[:, :3], 1, g)
    np.testing.assert_array_equal(res.state.rn_assignments, rn)


def test_zero_iterations_returns_exact_initial_layout():
    from paper_2303_05455_b200 import synth

    nb = synth.planted_graph(3000, 2, seed=2)
    res = P.run_embedding(graph=P.KnnGraph(nb), config=P.EmbeddingConfig(nn=2, rn=1, iterations=0, seed=8))
    np.testing.assert_array_equal(res.embedding.points, init_layout(3000, 2, np.random.default_rng(8)))
