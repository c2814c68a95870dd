"""The opt-in shim that routes the reference package's own callers (CLI,
steering server, operators, kNN, metrics) through this package
(paper_2303_05455_b200/reference_shim.py).  CPU test: it
imports the reference from /root/reference (present where the CPU suite runs;
skipped elsewhere) and checks the wiring — after `install` the reference CLI's
`embed` reaches this package's run_embedding (on a machine without a GPU the
call fails with this package's DeviceError, which the CLI reports), and
`uninstall` restores the reference."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def ivhd():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present")
    sys.path.insert(0, REF)
    try:
        import ivhd as mod
        import ivhd.cli  # noqa: F401
    except Exception as e:  # missing optional dependency of the reference
        pytest.skip(f"reference not importable: {e}")
    finally:
        sys.path.remove(REF)
    return mod


def test_install_routes_the_reference_entry_points(ivhd):
    import paper_2303_05455_b200 as P
    from paper_2303_05455_b200 import knng, metrics, reference_shim

    saved = reference_shim.install(ivhd)
    try:
        assert ivhd.engine.run_embedding is P.run_embedding
        assert ivhd.cli.run_embedding is P.run_embedding
        assert ivhd.forces.compute_forces is P.compute_forces
        assert ivhd.forces.stress is P.stress
        assert ivhd.knng.build_exact_knn is knng.build_exact_knn
        for name in ("neighbor_hit", "rnx_curve", "gnn_curve", "trust_continuity", "evaluate_embedding"):
            assert getattr(ivhd.metrics, name) is getattr(metrics, name)
    finally:
        reference_shim.uninstall(saved)
    assert ivhd.engine.run_embedding is not P.run_embedding
    assert ivhd.cli.run_embedding is ivhd.engine.run_embedding


def test_reference_cli_embed_reaches_this_package(ivhd, tmp_path):
    from click.testing import CliRunner

    import paper_2303_05455_b200 as P
    from paper_2303_05455_b200 import reference_shim

    rng = np.random.default_rng(0)
    m = 300
    nb = ((np.arange(m)[:, None] + rng.integers(1, 20, size=(m, 2))) % m).astype(np.int32)
    gpath = str(tmp_path / "g.ivhg")
    ivhd.knng.cache_write(ivhd.knng.KnnGraph(neighbors=nb, distances=np.ones(nb.shape), metric="euclidean"), gpath)
    calls = []
    real = P.run_embedding

    def recording(*a, **k):  # this package's entry point, observed
        calls.append(k)
        return real(*a, **k)

    saved = reference_shim.install(ivhd)
    ivhd.cli.run_embedding = recording  # stands in for P.run_embedding as installed
    try:
        res = CliRunner().invoke(ivhd.cli.main, ["embed", "--graph", gpath, "--out-dir", str(tmp_path / "out"),
                                                 "--iterations", "3", "--nn", "2"])
    finally:
        reference_shim.uninstall(saved)
    assert len(calls) == 1
    cfg = calls[0]["config"]
    assert (cfg.nn, cfg.iterations) == (2, 3) and calls[0]["graph"].neighbors.shape == (m, 2)
    try:
        import torch

        gpu = torch.cuda.is_available()
    except Exception:
        gpu = False
    if gpu:
        assert res.exit_code == 0, res.output
        assert os.path.exists(tmp_path / "out" / "embedding.csv")
    else:  # no GPU: this package's DeviceError — reported by the reference CLI when
        # it subclasses ivhd.errors.IvhdError (this package imported after ivhd),
        # raised through otherwise
        assert res.exit_code != 0
        assert isinstance(res.exception, P.DeviceError) or (
            "DeviceError" in res.output and "ivhd status" in res.output), (res.output, res.exception)
