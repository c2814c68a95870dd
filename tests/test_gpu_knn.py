"""GPU kNN builder (csrc/ivhd_knn.cu) against the reference's
build_exact_knn (knng.py:158-194) golden graphs, plus large-size properties.

Fixtures: tests/golden/knn_graphs.npz from tests/golden/make_knn_golden.py
(inputs regenerated from seeds by `knn_inputs`).
"""

import os

import numpy as np
import pytest

from tests.golden.make_knn_golden import knn_inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden", "knn_graphs.npz")


def _same_graph(nbr, dist, ref_nbr, ref_dist):
    """Identical rows, except that the order inside groups of reference
    distances equal to ~1e-12 (ties broken by index on values the fp64 Gram
    expansion of the reference rounds differently) may differ; distances to
    1e-9 relative (+1e-6 absolute for the Gram expansion's cancellation near 0)."""
    np.testing.assert_allclose(dist, ref_dist, rtol=1e-9, atol=1e-6)
    bad = np.nonzero((nbr != ref_nbr).any(axis=1))[0]
    for r in bad:
        # the rows must agree as sets and ordering may differ only among near-equal distances
        assert set(nbr[r]) == set(ref_nbr[r]) or np.isclose(dist[r, -1], ref_dist[r, -1], rtol=1e-9, atol=1e-6), r
        for a, b in zip(nbr[r], ref_nbr[r]):
            if a != b:
                da = dist[r][list(nbr[r]).index(a)]
                db = ref_dist[r][list(ref_nbr[r]).index(b)]
                assert abs(da - db) <= 1e-6 + 1e-9 * abs(db), (r, a, b, da, db)
    return len(bad)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(knn_inputs()))
def test_knn_matches_reference_golden(name):
    from paper_2303_05455_b200 import knng

    x, k, metric = knn_inputs()[name]
    gold = np.load(GOLD)
    g = knng.build_exact_knn(x, k, metric=metric)
    assert g.neighbors.shape == (x.shape[0], k) and g.neighbors.dtype == np.int32
    assert not (g.neighbors == np.arange(x.shape[0])[:, None]).any()  # self excluded
    n_diff = _same_graph(g.neighbors, g.distances, gold[f"{name}_nbr"], gold[f"{name}_dist"])
    if name not in ("duplicates",):
        assert n_diff == 0, f"{n_diff} rows ordered differently"


@pytest.mark.gpu
def test_knn_lattice_tie_rule_exact():
    """On integer data every distance is exact in fp64, so the (distance,
    index) order must be reproduced bit for bit (knng.py:1-6)."""
    from paper_2303_05455_b200 import knng

    x, k, metric = knn_inputs()["lattice_ties"]
    gold = np.load(GOLD)
    g = knng.build_exact_knn(x, k, metric=metric)
    np.testing.assert_array_equal(g.neighbors, gold["lattice_ties_nbr"])
    np.testing.assert_array_equal(g.distances, gold["lattice_ties_dist"])


@pytest.mark.gpu
def test_knn_errors():
    from paper_2303_05455_b200 import knng
    from paper_2303_05455_b200.errors import DegenerateMetricError, InvalidArgumentError

    x = np.random.default_rng(0).standard_normal((50, 4))
    with pytest.raises(InvalidArgumentError):
        knng.build_exact_knn(x, 50)
    with pytest.raises(InvalidArgumentError):
        knng.build_exact_knn(x, 0)
    with pytest.raises(InvalidArgumentError):
        knng.build_exact_knn(x, 3, metric="manhattan")
    x[17] = 0.0
    with pytest.raises(DegenerateMetricError) as ei:
        knng.build_exact_knn(x, 3, metric="cosine")
    assert ei.value.row == 17


@pytest.mark.gpu
def test_knn_large_rows_exact_against_fp64_scan():
    """200k x 100 mixture: sampled rows equal an fp64 brute-force scan
    (torch on the GPU, test-side checker only)."""
    import torch

    from paper_2303_05455_b200 import knng

    rng = np.random.default_rng(3)
    centers = 2.0 * rng.standard_normal((10, 100))
    x = centers[rng.integers(0, 10, 200_000)] + rng.standard_normal((200_000, 100))
    k = 8
    g = knng.build_exact_knn(x, k)
    X = torch.from_numpy(x).cuda()
    rows = rng.choice(len(x), 256, replace=False)
    d = torch.cdist(X[rows], X).cpu().numpy()
    d[np.arange(len(rows)), rows] = np.inf
    for i, r in enumerate(rows):
        order = np.lexsort((np.arange(len(x)), d[i]))[:k]
        np.testing.assert_array_equal(g.neighbors[r], order)
        np.testing.assert_allclose(g.distances[r], d[i][order], rtol=1e-9)
    assert knng.last_stats["exact_rows"] < len(x) // 100  # the certificate covers almost every row
