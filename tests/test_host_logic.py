"""Host-side logic of the drop-in (no GPU): configuration, seeded set-up
draws, RNN filter, mutations, trace, errors, shard planning."""

import json
import os
import warnings

import numpy as np
import pytest

import oracle as O
import paper_2303_05455_b200 as P
from paper_2303_05455_b200 import config as C
from paper_2303_05455_b200.embed import _apply_mutation
from paper_2303_05455_b200.sharded import shard_ranges

from .conftest import GOLDEN

BLOB = np.load(os.path.join(GOLDEN, "blob_graph.npz"))
META = json.load(open(os.path.join(GOLDEN, "meta.json")))


class TestConfig:
    # mirrors the reference's test_engine.py:141-169 validation cases
    def test_c_range(self):
        with pytest.raises(P.InvalidArgumentError):
            P.EmbeddingConfig(c=0.0)
        with pytest.raises(P.InvalidArgumentError):
            P.EmbeddingConfig(c=1.0)

    def test_phase_budget(self):
        with pytest.raises(P.InvalidArgumentError):
            P.EmbeddingConfig(iterations=100, l1_final_steps=200)

    def test_nn_rn_warning(self):
        with pytest.warns(UserWarning, match="long-range"):
            P.EmbeddingConfig(nn=1, rn=2)

    @pytest.mark.parametrize("kw", [dict(nn=0), dict(rn=0), dict(target_dim=4), dict(iterations=-1),
                                    dict(optimizer="bfgs"), dict(distance_mode="cosine"),
                                    dict(rn_resample_period=-1), dict(rnn_final_steps=-1)])
    def test_rejects(self, kw):
        with pytest.raises(P.InvalidArgumentError):
            P.EmbeddingConfig(**kw)

    def test_roundtrip_dict(self):
        cfg = P.EmbeddingConfig(nn=4, rn=2, c=0.05, optimizer="adam")
        back = P.EmbeddingConfig.from_dict(cfg.to_dict())
        assert back.to_dict() == cfg.to_dict()
        assert isinstance(back.integrator, P.IntegratorParams)

    def test_integrator(self):
        with pytest.raises(P.InvalidArgumentError):
            P.IntegratorParams(a=1.5)
        with pytest.raises(P.InvalidArgumentError):
            P.IntegratorParams(b=0.0)
        with pytest.raises(P.InvalidArgumentError):
            P.IntegratorParams(gamma1=0.9)
        p = P.IntegratorParams.from_physics(0.3, 0.1, 2.0)
        assert p.a / p.b == pytest.approx((1 - 0.015) / (2 * 2.0 * 0.1), rel=1e-12)
        assert P.IntegratorParams().tau_for(2000) == pytest.approx(2.0)

    def test_resolve_optimizer(self):
        p = C.resolve_optimizer("force-directed", 1000)
        assert p.kind == 0 and p.step == 0.002 and p.tau == pytest.approx(1.0) and p.auto_adapt == 1
        for kind, alpha in C.DEFAULT_ALPHA.items():
            assert C.resolve_optimizer(kind, 10).step == alpha
        assert C.resolve_optimizer("adam", 10, opt=P.OptimizerParams(alpha=0.3)).step == 0.3
        with pytest.raises(P.InvalidArgumentError):
            C.resolve_optimizer("lbfgs", 10)


class TestSeededDraws:
    """Y0 and rn are bit-identical to the reference's (engine.py:124-146)."""

    @pytest.mark.parametrize("name", sorted(k for k in META if k.startswith("replay_")))
    def test_matches_reference_golden(self, name):
        meta = META[name]
        g = np.load(os.path.join(GOLDEN, name + ".npz"))
        rng = np.random.default_rng(meta["seed"])
        y0 = P.init_layout(BLOB["neighbors"].shape[0], meta["target_dim"], rng)
        rn = P.sample_random_neighbors(y0.shape[0], BLOB["neighbors"][:, :meta["nn"]], meta["rn"], rng)
        np.testing.assert_array_equal(y0, g["Y0"])
        np.testing.assert_array_equal(rn, g["rn"])

    def test_forced_choice_and_exclusion(self):
        assert P.sample_random_neighbors(3, np.array([[1], [2], [0]]), 1, seed=0).ravel().tolist() == [2, 0, 1]
        with pytest.raises(P.InvalidArgumentError):
            P.sample_random_neighbors(3, np.array([[1], [2], [0]]), 2, seed=0)
        rng = np.random.default_rng(1)
        nn = np.argsort(rng.standard_normal((200, 200)), axis=1)[:, :5]
        a = P.sample_random_neighbors(200, nn, 3, seed=2)
        for i in range(200):
            assert i not in a[i] and not set(a[i]) & set(nn[i])

    def test_matches_oracle(self):
        nb = BLOB["neighbors"][:, :3]
        a = P.sample_random_neighbors(nb.shape[0], nb, 2, np.random.default_rng(5))
        b = O.sample_rn(nb.shape[0], nb, 2, np.random.default_rng(5))
        np.testing.assert_array_equal(a, b)

    def test_init_layout(self):
        y = P.init_layout(1000, 3, 3)
        assert y.shape == (1000, 3) and y.min() >= -1 and y.max() <= 1
        with pytest.raises(P.InvalidArgumentError):
            P.init_layout(0, 2, 0)


def test_rnn_filter_matches_oracle():
    nb = BLOB["neighbors"]
    m = nb.shape[0]
    nn = nb[:, :2]
    edges = np.column_stack([np.repeat(np.arange(m), 2), nn.ravel()])
    keep = P.rnn_edge_filter(edges, nn, P.KnnGraph(nb))
    ref = O.rnn_keep_mask(edges[:, 0], edges[:, 1], nn, nb)
    np.testing.assert_array_equal(keep, ref)
    assert keep.reshape(m, 2).any(axis=1).all()


class _Sess:
    def __init__(self, kind="force-directed"):
        self.c = 0.1
        self.config = P.EmbeddingConfig(optimizer=kind)
        self.calls = []

        class Dev:
            def set_step_size(dev, v):
                self.calls.append(("b", v))

        self.dev = Dev()

    def set_optimizer(self, kind):
        self.calls.append(("optimizer", kind))


class TestMutations:
    """engine.py:417-448 semantics, including the Adadelta 'b' quirk."""

    def test_c(self):
        s = _Sess()
        assert _apply_mutation(s, "c", 0.02) == 0.02 and s.c == 0.02
        with pytest.raises(P.InvalidArgumentError):
            _apply_mutation(s, "c", 42.0)

    def test_b(self):
        s = _Sess()
        assert _apply_mutation(s, "b", 0.5) == 0.5
        assert s.calls == [("b", 0.5)]
        with pytest.raises(P.InvalidArgumentError):
            _apply_mutation(s, "b", -1)
        s = _Sess("adadelta")  # the reference's Adadelta has neither params.b nor alpha
        assert _apply_mutation(s, "b", 0.5) == 0.5 and s.calls == []

    def test_other_keys(self):
        s = _Sess()
        assert _apply_mutation(s, "optimizer", "adam") == "adam" and s.calls == [("optimizer", "adam")]
        with pytest.raises(P.InvalidArgumentError):
            _apply_mutation(s, "optimizer", "bfgs")
        assert _apply_mutation(s, "rn_resample_period", "3") == 3
        with pytest.raises(P.InvalidArgumentError):
            _apply_mutation(s, "rn_resample_period", -2)
        assert _apply_mutation(s, "stop", 1) is True
        with pytest.raises(P.InvalidArgumentError):
            _apply_mutation(s, "nonsense", 1)


def test_trace_csv(tmp_path):
    tr = P.StressTrace()
    tr.extend(0, [1.5, 2.25], [0.002, 0.0018])
    tr.append(2, 3.0, 0.001)
    p = tmp_path / "t.csv"
    tr.to_csv(str(p))
    lines = p.read_text().strip().splitlines()
    assert lines[0] == "iteration,stress,b" and len(lines) == 4
    assert lines[2] == "1,2.25,0.0018"


def test_errors_hierarchy():
    err = P.NumericalDivergenceError(7, state="s")
    assert isinstance(err, P.IvhdError) and err.iteration == 7 and err.state == "s"
    assert issubclass(P.InvalidArgumentError, P.IvhdError)
    import os
    import subprocess
    import sys

    if not os.path.isdir("/root/reference/pkg/src"):  # build container only
        return
    # with the reference importable, callers catching its classes keep working
    # (fresh interpreter: reloading the module here would swap the classes
    # under the other tests' feet)
    code = ("import sys; sys.path.insert(0, '/root/reference/pkg/src'); import ivhd.errors as ref; "
            "from paper_2303_05455_b200 import errors as E; "
            "assert issubclass(E.InvalidArgumentError, ref.InvalidArgumentError); "
            "assert issubclass(E.MalformedInputError, ref.MalformedInputError); "
            "assert issubclass(E.DegenerateMetricError, ref.DegenerateMetricError)")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_embedding_and_graph_types():
    with pytest.raises(P.DimensionMismatchError):
        P.Embedding(np.zeros((3, 4)))
    g = P.KnnGraph([[1, 2], [0, 2], [0, 1]], np.ones((3, 2)))
    assert g.M == 3 and g.k == 2 and g.neighbors.dtype == np.int32
    with pytest.raises(P.DimensionMismatchError):
        P.KnnGraph([[1, 2], [0, 2]], np.ones((2, 3)))


def test_graph_or_dataset_required():
    with pytest.raises(P.InvalidArgumentError):
        P.run_embedding(graph=None, config=P.EmbeddingConfig(iterations=1))


def test_shard_ranges():
    r = shard_ranges(16, 256, 4)
    assert r == [(0, 1024), (1024, 2048), (2048, 3072), (3072, 4096)]
    with pytest.raises(P.InvalidArgumentError):
        shard_ranges(12, 256, 8)
