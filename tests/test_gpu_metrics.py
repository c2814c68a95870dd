"""GPU neighbour hit (csrc/ivhd_metrics.cu) against the reference's
metrics.neighbor_hit golden curves (tests/golden/make_metrics_golden.py) and
against scipy's cKDTree at scale."""

import os

import numpy as np
import pytest

from tests.golden.make_metrics_golden import metric_inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden", "neighbor_hit.npz")


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(metric_inputs()))
def test_neighbor_hit_matches_reference(name):
    from paper_2303_05455_b200 import metrics

    y, lab, k = metric_inputs()[name]
    cf_nn, cf = metrics.neighbor_hit(y, lab, nn_max=k)
    ref = np.load(GOLD)[name]
    # exact kNN on both sides: equal curves (ties of equal-label points cannot
    # change a count; the reference's M > 20000 branch uses a k-d tree whose
    # tie order is arbitrary, so allow one tie flip per size there)
    tol = 0.0 if "30k" not in name else 1.0 / (len(y))
    np.testing.assert_allclose(cf_nn, ref, rtol=0, atol=tol + 1e-15)
    assert cf == pytest.approx(float(ref.mean()), abs=tol + 1e-15)


@pytest.mark.gpu
def test_neighbor_hit_graph_input_and_errors():
    from paper_2303_05455_b200 import metrics
    from paper_2303_05455_b200.embed import KnnGraph
    from paper_2303_05455_b200.errors import InvalidArgumentError

    y, lab, k = metric_inputs()["blobs2d_4k"]
    cf_nn, cf, nbr = metrics.neighbor_hit(y, lab, nn_max=k, return_neighbors=True)
    g_nn, g_cf = metrics.neighbor_hit(KnnGraph(nbr), lab, nn_max=k)
    np.testing.assert_allclose(g_nn, cf_nn, rtol=0, atol=1e-15)
    with pytest.raises(InvalidArgumentError):
        metrics.neighbor_hit(y, lab, nn_max=len(y))
    with pytest.raises(InvalidArgumentError):
        metrics.neighbor_hit(y, None)


@pytest.mark.gpu
def test_neighbor_ids_equal_kdtree_at_scale():
    """300k 2-D points: every neighbour list equals scipy's cKDTree query
    (continuous coordinates: no ties)."""
    from scipy.spatial import cKDTree

    from paper_2303_05455_b200 import metrics

    rng = np.random.default_rng(5)
    c = rng.uniform(-10, 10, (12, 2))
    lab = rng.integers(0, 12, 300_000)
    y = c[lab] + rng.standard_normal((300_000, 2)) * rng.uniform(0.2, 2.0, (300_000, 1))
    cf_nn, cf, nbr = metrics.neighbor_hit(y, lab, nn_max=100, return_neighbors=True)
    rows = rng.choice(len(y), 2000, replace=False)
    _, idx = cKDTree(y).query(y[rows], k=101)
    np.testing.assert_array_equal(nbr[rows], idx[:, 1:])


# ------------------------------------------------------------- rank curves
from tests.golden.make_curves_golden import OUT as CURVES_GOLD, curve_inputs  # noqa: E402


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(curve_inputs()))
def test_evaluate_embedding_matches_reference(name):
    """GPU curve pass (ivhd_curve_pass) against the reference's
    evaluate_embedding.  Ranks come from fp64 distances summed in a different
    order than the reference's BLAS, so a near-tie may flip: each curve value
    is an average of integer counts over k*M pairs; allow a few flips."""
    from paper_2303_05455_b200 import metrics

    X, Y, lab, k_max, ks, pre = curve_inputs()[name]
    gold = np.load(CURVES_GOLD)
    cur = metrics.evaluate_embedding(X, Y, labels=lab, k_max=k_max, nn_max=20, report_ks=ks, x_precomputed=pre)
    m = len(Y)
    exact = "lattice" in name or "precomp" in name  # integer arithmetic / given distances
    tol = 0.0 if exact else 4.0 / m
    np.testing.assert_allclose(cur.q_nx, gold[f"{name}/q_nx"], rtol=0, atol=tol + 1e-15)
    np.testing.assert_allclose(cur.r_nx, gold[f"{name}/r_nx"], rtol=0, atol=2 * tol + 1e-15)
    assert cur.auc_rnx == pytest.approx(float(gold[f"{name}/auc_rnx"]), abs=tol + 1e-15)
    if lab is not None:
        np.testing.assert_allclose(cur.g_nn, gold[f"{name}/g_nn"], rtol=0, atol=tol + 1e-15)
        assert cur.auc_gnn == pytest.approx(float(gold[f"{name}/auc_gnn"]), abs=tol + 1e-15)
    keep = [k for k in ks if k < m / 2]
    np.testing.assert_allclose([cur.trust[k] for k in keep], gold[f"{name}/trust"], rtol=0, atol=tol + 1e-15)
    np.testing.assert_allclose([cur.continuity[k] for k in keep], gold[f"{name}/continuity"], rtol=0,
                               atol=tol + 1e-15)
    if not pre:
        _, _, _, auc = metrics.rnx_curve(X, Y, k_max=k_max)
        assert auc == pytest.approx(float(gold[f"{name}/rnx_auc_direct"]), abs=tol + 1e-15)
        t, c = metrics.trust_continuity(X, Y, ks[0])
        np.testing.assert_allclose([t, c], gold[f"{name}/tc_direct"], rtol=0, atol=tol + 1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1])
def test_curve_counts_equal_oracle(seed):
    """Integer counts equal the oracle restatement (metrics.py:149-182) on
    integer-valued inputs (exact distances, heavy ties)."""
    import oracle as O
    from paper_2303_05455_b200 import metrics

    rng = np.random.default_rng(100 + seed)
    m = 700 + 37 * seed
    X = rng.integers(-4, 5, (m, 6)).astype(np.float64)
    Y = rng.integers(-6, 7, (m, 2 + seed)).astype(np.float64)
    lab = rng.integers(0, 5, m)
    ks = (3, 20, 100)
    got = metrics._curve_pass(X, Y, lab, 300, ks)
    want = O.curve_pass(X, Y, lab, 300, ks)
    for g, w in zip(got[:3], want[:3]):
        np.testing.assert_array_equal(g, w)
    assert got[3] == want[3] and got[4] == want[4]


@pytest.mark.gpu
def test_curves_identity_embedding_at_scale():
    """Size-independent property at C1 scale (M=20000, several distance
    blocks): an embedding equal to the source ranks every pair identically,
    so Q_NX = R_NX = 1, trust = continuity = 1 and G_NN = 0."""
    from paper_2303_05455_b200 import metrics

    rng = np.random.default_rng(7)
    m = 20000
    X = rng.standard_normal((m, 2)) * np.array([3.0, 1.0])
    lab = (X[:, 0] > 0).astype(np.int64)
    cur = metrics.evaluate_embedding(X, X.copy(), labels=lab, report_ks=(15, 100))
    np.testing.assert_array_equal(cur.q_nx, np.ones(1000))
    assert cur.auc_rnx == pytest.approx(1.0, abs=1e-12)
    np.testing.assert_array_equal(cur.g_nn, np.zeros(1000))
    assert cur.trust == {15: 1.0, 100: 1.0} and cur.continuity == {15: 1.0, 100: 1.0}


@pytest.mark.gpu
def test_curve_errors():
    from paper_2303_05455_b200 import metrics
    from paper_2303_05455_b200.errors import DimensionMismatchError, InvalidArgumentError

    X = np.random.default_rng(0).standard_normal((50, 4))
    with pytest.raises(InvalidArgumentError):
        metrics.rnx_curve(X, X[:, :2], k_max=49)
    with pytest.raises(DimensionMismatchError):
        metrics.rnx_curve(X, X[:40, :2])
    with pytest.raises(InvalidArgumentError):
        metrics.gnn_curve(X, X[:, :2], None)
    with pytest.raises(InvalidArgumentError):
        metrics.trust_continuity(X, X[:, :2], 25)
    with pytest.raises(InvalidArgumentError):
        metrics.rnx_curve(X[:3], X[:3, :2])


@pytest.mark.gpu
def test_curve_counts_tie_crowded_rows_equal_oracle():
    """Rows whose K-th distance is shared by > 1000 points (3000 points on 4
    embedded locations) take the merge fallback of the radix select; counts
    still equal the oracle's (index tie rule)."""
    import oracle as O
    from paper_2303_05455_b200 import metrics

    rng = np.random.default_rng(9)
    m = 3000
    X = rng.integers(0, 3, (m, 4)).astype(np.float64)
    Y = rng.integers(0, 2, (m, 2)).astype(np.float64)
    lab = rng.integers(0, 3, m)
    got = metrics._curve_pass(X, Y, lab, 1000, (10, 100))
    want = O.curve_pass(X, Y, lab, 1000, (10, 100))
    for g, w in zip(got[:3], want[:3]):
        np.testing.assert_array_equal(g, w)
    assert got[3] == want[3] and got[4] == want[4]


@pytest.mark.gpu
@pytest.mark.parametrize("name", [n for n in sorted(curve_inputs()) if not curve_inputs()[n][5]])
def test_shepard_and_corank_matches_reference(name):
    """GPU pair ranks (ivhd_pair_ranks) against the reference's
    shepard_and_corank on the same sampled pairs: exact on integer inputs,
    at most 1% of ranks differing (near-ties under another fp64 summation
    order) otherwise."""
    from paper_2303_05455_b200 import metrics

    X, Y, _, _, _, _ = curve_inputs()[name]
    gold = np.load(CURVES_GOLD)
    (dl, _), (rho, r), r2 = metrics.shepard_and_corank(X, Y, sample_pairs=min(3000, len(Y) * 4), seed=3)
    np.testing.assert_array_equal(dl, gold[f"{name}/shepard_deltas"])
    if "lattice" in name:
        np.testing.assert_array_equal(rho, gold[f"{name}/shepard_rho"])
        np.testing.assert_array_equal(r, gold[f"{name}/shepard_r"])
        assert r2 == float(gold[f"{name}/shepard_r2"])
    else:
        assert np.mean(rho != gold[f"{name}/shepard_rho"]) <= 0.01
        assert np.mean(r != gold[f"{name}/shepard_r"]) <= 0.01
        assert r2 == pytest.approx(float(gold[f"{name}/shepard_r2"]), abs=1e-3)


@pytest.mark.gpu
def test_pair_ranks_equal_bruteforce_at_scale():
    """70k x 50 points, 5000 pairs (several distance blocks): ranks equal a
    numpy count over the same formula for a subset of pairs."""
    from paper_2303_05455_b200 import metrics

    rng = np.random.default_rng(4)
    m = 70000
    Z = rng.integers(-3, 4, (m, 5)).astype(np.float64)  # integer: exact distances, many ties
    (_, _), (rho, _), _ = metrics.shepard_and_corank(Z, Z[:, :2], sample_pairs=5000, seed=1)
    flat = np.random.default_rng(1).choice(m * (m - 1) // 2, size=5000, replace=False)
    i_idx, j_idx = metrics._unrank_pairs(flat, m)
    sq = (Z * Z).sum(1)
    for p in range(0, 5000, 250):
        i, j = i_idx[p], j_idx[p]
        row = np.maximum(sq[i] + sq - 2.0 * (Z @ Z[i]), 0.0)
        row[i] = np.inf
        want = 1 + np.count_nonzero(row < row[j]) + np.count_nonzero((row == row[j]) & (np.arange(m) < j))
        assert rho[p] == want


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["lattice_400_ties", "precomp_300", "tiny_40", "mix20_600"])
def test_compute_ranks_equal_oracle(name):
    """GPU rank matrix vs the oracle restatement of metrics.py:103-113 (exact on
    integer / given distances; near-ties may swap neighbours otherwise)."""
    import oracle as O
    from paper_2303_05455_b200 import metrics

    X, Y, _, _, _, pre = curve_inputs()[name]
    if pre:
        rd = metrics.compute_ranks(distances=X, ld_distances=X[::-1, ::-1])
        want_hd = O.ivhd_oracle._ranks(X)[0]
        want_ld = O.ivhd_oracle._ranks(np.ascontiguousarray(X[::-1, ::-1]))[0]
        np.testing.assert_array_equal(rd.ld_ranks, want_ld)
    else:
        rd = metrics.compute_ranks(dataset=X)
        want_hd = O.ivhd_oracle._ranks(O.ivhd_oracle._sq_dist_matrix(X))[0]
        assert rd.ld_ranks is None
    if "mix" in name:
        assert np.mean(rd.hd_ranks != want_hd) < 1e-3
    else:
        np.testing.assert_array_equal(rd.hd_ranks, want_hd)
    m = len(X)
    assert (np.diag(rd.hd_ranks) == 0).all()
    np.testing.assert_array_equal(np.sort(rd.hd_ranks, axis=1), np.broadcast_to(np.arange(m), (m, m)))


@pytest.mark.gpu
def test_compute_ranks_blocks_and_errors():
    """9000 points: several row blocks; rows are permutations of 0..M-1."""
    from paper_2303_05455_b200 import metrics
    from paper_2303_05455_b200.errors import DimensionMismatchError, InvalidArgumentError

    X = np.random.default_rng(2).integers(0, 5, (9000, 3)).astype(np.float64)
    r = metrics.compute_ranks(dataset=X).hd_ranks
    assert (np.diag(r) == 0).all()
    for i in (0, 4321, 8999):
        row = np.maximum((X * X).sum(1)[i] + (X * X).sum(1) - 2.0 * (X @ X[i]), 0.0)
        row[i] = np.inf
        order = np.lexsort((np.arange(9000), row))
        want = np.empty(9000, dtype=np.int64)
        want[order] = np.arange(1, 9001)
        want[i] = 0
        np.testing.assert_array_equal(r[i], want)
    with pytest.raises(InvalidArgumentError):
        metrics.compute_ranks()
    with pytest.raises(DimensionMismatchError):
        metrics.compute_ranks(distances=np.zeros((3, 4)))
    with pytest.raises(InvalidArgumentError):
        metrics.compute_ranks(dataset=np.zeros((1, 2)))


@pytest.mark.gpu
def test_many_report_ks_take_extra_passes():
    """More report ks than one device pass holds (8): same values as one k at a time."""
    from paper_2303_05455_b200 import metrics

    X, Y, lab, _, _, _ = curve_inputs()["mix20_600"]
    ks = tuple(range(5, 290, 25))  # 12 ks
    cur = metrics.evaluate_embedding(X, Y, labels=lab, k_max=50, nn_max=10, report_ks=ks)
    assert sorted(cur.trust) == list(ks)
    for k in (5, 205, 280):
        t, c = metrics.trust_continuity(X, Y, k)
        assert cur.trust[k] == t and cur.continuity[k] == c


@pytest.mark.gpu
@pytest.mark.parametrize("k", [129, 300, 512])
def test_neighbor_hit_large_nn_max_equals_kdtree(k):
    """nn_max above 128 (8 / 16 slots per lane): neighbour ids equal scipy's
    cKDTree on continuous 2-D points, and the hit curve follows from them."""
    from scipy.spatial import cKDTree

    from paper_2303_05455_b200 import metrics

    rng = np.random.default_rng(k)
    y = rng.standard_normal((6000, 2))
    lab = (y[:, 0] > 0).astype(np.int64) + 2 * (y[:, 1] > 0.3)
    cf_nn, cf, nbr = metrics.neighbor_hit(y, lab, nn_max=k, return_neighbors=True)
    _, idx = cKDTree(y).query(y, k=k + 1)
    np.testing.assert_array_equal(nbr, idx[:, 1:])
    same = lab[idx[:, 1:]] == lab[:, None]
    want = same.cumsum(axis=1).sum(axis=0) / (np.arange(1, k + 1) * len(y))
    np.testing.assert_allclose(cf_nn, want, rtol=0, atol=1e-15)
