"""Embedding quality metrics on the GPU.

Rank curves: `rnx_curve`, `gnn_curve`, `trust_continuity` and
`evaluate_embedding` are drop-ins for the reference's functions of the same
names (metrics.py:185-251, 351-380).  Their counts come from one GPU pass
(`ivhd_curve_pass`, csrc/ivhd_metrics.cu) that replaces the reference's
streamed `_curve_pass` (metrics.py:149-182).  The host arithmetic on those
integer counts (`_curves_from_counts`, `_gnn_from_counts`, `_unrank_pairs`, the
trust / continuity scaling, and the body of `shepard_and_corank` /
`evaluate_embedding`) is the reference's arithmetic kept verbatim
(metrics.py:208-236, 297-320, 323-332, 355-385), so the golden tests can demand
bit-identical floating-point results on identical counts; the GPU code is what
produces the counts.

`neighbor_hit` is the drop-in for the reference's `ivhd.metrics.neighbor_hit`
(/root/reference/pkg/src/ivhd/metrics.py:254-294): same signature, same
(cf_nn, cf) result.  For embedded points the nn_max nearest neighbours come
from the exact grid kNN in csrc/ivhd_metrics.cu (2-D/3-D); for a prebuilt
KnnGraph the reference's arithmetic on the given neighbour block is applied
directly (label comparisons only, no search).
"""

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import DeviceError, DimensionMismatchError, InvalidArgumentError


def neighbor_hit(y_or_graph, labels, nn_max=100, device=0, return_neighbors=False):
    if labels is None:
        raise InvalidArgumentError("neighbor hit needs class labels")
    labels = np.asarray(labels)
    if hasattr(y_or_graph, "neighbors"):  # KnnGraph (metrics.py:271-278)
        graph = y_or_graph
        if graph.neighbors.shape[1] < nn_max:
            raise InvalidArgumentError(f"graph stores {graph.neighbors.shape[1]} neighbors, need nn_max={nn_max}")
        nbrs = np.asarray(graph.neighbors)[:, :nn_max]
        if labels.shape[0] != nbrs.shape[0]:
            raise DimensionMismatchError("labels and points row counts differ")
        same = labels[nbrs] == labels[:, None]
        per_size = same.cumsum(axis=1).sum(axis=0)
        cf_nn = per_size / (np.arange(1, nn_max + 1) * labels.shape[0])
        return cf_nn, float(cf_nn.mean())
    y = np.asarray(y_or_graph, dtype=np.float64)
    if y.ndim == 1:
        y = y[:, None]
    m = y.shape[0]
    if not (1 <= nn_max < m):
        raise InvalidArgumentError(f"nn_max must be in [1, M), got {nn_max}")
    if labels.shape[0] != m:
        raise DimensionMismatchError("labels and points row counts differ")
    # labels of any type -> dense int32 codes (equality is all that matters)
    _, codes = np.unique(labels, return_inverse=True)
    codes = np.ascontiguousarray(codes.reshape(-1), dtype=np.int32)
    y = np.ascontiguousarray(y)
    lib = _lib.load()
    cf_nn = np.empty(nn_max, dtype=np.float64)
    nbr = np.empty((m, nn_max), dtype=np.int32) if return_neighbors else None
    rc = lib.ivhd_neighbor_hit(int(device), _lib.ptr(y, _lib.ctypes.c_double), m, int(y.shape[1]),
                               _lib.ptr(codes, _lib.ctypes.c_int32), int(nn_max),
                               _lib.ptr(cf_nn, _lib.ctypes.c_double), _lib.ptr(nbr, _lib.ctypes.c_int32))
    if rc != _lib.OK:
        msg = (lib.ivhd_metrics_last_error() or b"").decode(errors="replace")
        if rc == _lib.ERR_INVALID_ARG:
            raise InvalidArgumentError(msg)
        raise DeviceError(f"neighbor_hit failed: {msg}")
    if return_neighbors:
        return cf_nn, float(cf_nn.mean()), nbr
    return cf_nn, float(cf_nn.mean())


# ------------------------------------------------------------------ rank curves


@dataclass
class MetricCurves:
    """Per-k quality curves plus scalar summaries (reference metrics.py:26-53)."""

    k: np.ndarray
    q_nx: np.ndarray
    r_nx: np.ndarray
    auc_rnx: float
    g_nn: np.ndarray | None = None
    auc_gnn: float | None = None
    trust: dict = field(default_factory=dict)
    continuity: dict = field(default_factory=dict)
    cf_nn: np.ndarray | None = None
    cf: float | None = None

    def summary(self):
        out = {"auc_rnx": self.auc_rnx}
        if self.auc_gnn is not None:
            out["auc_gnn"] = self.auc_gnn
        if self.cf is not None:
            out["cf"] = self.cf
            for probe in (2, 10, 100):
                if self.cf_nn is not None and probe <= len(self.cf_nn):
                    out[f"cf_{probe}"] = float(self.cf_nn[probe - 1])
        for k, v in self.trust.items():
            out[f"trustworthiness_k{k}"] = v
        for k, v in self.continuity.items():
            out[f"continuity_k{k}"] = v
        return out


def _as_matrix(data):
    mat = np.asarray(getattr(data, "data", data), dtype=np.float64)
    if mat.ndim != 2:
        raise DimensionMismatchError(f"expected a 2-D matrix, got shape {mat.shape}")
    return mat


def default_k_max(m):
    return min(m - 2, 1000)


_MAX_REPORT = 8  # report ks per device pass (ivhd_curve_pass)


def _curve_pass(X, Y, labels, k_max, report_ks, x_precomputed=False, device=0):
    """GPU restatement of metrics.py:149-182: (agree[0..k_max], same_ld, same_hd,
    trust_pen, cont_pen).  agree is truncated at k_max, which is all the curves
    read (cumsum(agree)[1:k_max+1]).  More than 8 report ks take extra passes
    (trust/continuity only)."""
    report_ks = [int(k) for k in report_ks]
    if len(report_ks) > _MAX_REPORT:
        out = _curve_pass(X, Y, labels, k_max, report_ks[:_MAX_REPORT], x_precomputed, device)
        for a in range(_MAX_REPORT, len(report_ks), _MAX_REPORT):
            _, _, _, t, c = _curve_pass(X, Y, None, 1, report_ks[a:a + _MAX_REPORT], x_precomputed, device)
            out[3].update(t)
            out[4].update(c)
        return out
    m = X.shape[0]
    if Y.shape[0] != m:
        raise DimensionMismatchError("X and Y row counts differ")
    if x_precomputed and X.shape[1] != m:
        raise DimensionMismatchError("precomputed distances must be square")
    if not 1 <= Y.shape[1] <= 3:
        raise InvalidArgumentError(f"rank curves on the GPU need a 1-3 dimensional embedding, got {Y.shape[1]}")
    codes = None
    if labels is not None:
        labels = np.asarray(labels)
        if labels.shape[0] != m:
            raise DimensionMismatchError("labels and points row counts differ")
        _, codes = np.unique(labels, return_inverse=True)
        codes = np.ascontiguousarray(codes.reshape(-1), dtype=np.int32)
    ks = np.ascontiguousarray([int(k) for k in report_ks], dtype=np.int32)
    x = np.ascontiguousarray(X)
    y = np.ascontiguousarray(Y)
    agree = np.zeros(k_max + 1, dtype=np.int64)
    same_ld = np.zeros(k_max, dtype=np.int64)
    same_hd = np.zeros(k_max, dtype=np.int64)
    trust = np.zeros(max(len(ks), 1), dtype=np.int64)
    cont = np.zeros(max(len(ks), 1), dtype=np.int64)
    lib = _lib.load()
    c_i64 = _lib.ctypes.c_int64
    rc = lib.ivhd_curve_pass(int(device), _lib.ptr(x, _lib.ctypes.c_double), m, int(x.shape[1]), int(bool(x_precomputed)),
                             _lib.ptr(y, _lib.ctypes.c_double), int(y.shape[1]), _lib.ptr(codes, _lib.ctypes.c_int32),
                             int(k_max), _lib.ptr(ks, _lib.ctypes.c_int32), len(ks), _lib.ptr(agree, c_i64),
                             _lib.ptr(same_ld, c_i64), _lib.ptr(same_hd, c_i64), _lib.ptr(trust, c_i64),
                             _lib.ptr(cont, c_i64))
    if rc != _lib.OK:
        msg = (lib.ivhd_metrics_last_error() or b"").decode(errors="replace")
        if rc == _lib.ERR_INVALID_ARG:
            raise InvalidArgumentError(msg)
        raise DeviceError(f"curve pass failed: {msg}")
    trust_pen = {int(k): int(trust[a]) for a, k in enumerate(ks)}
    cont_pen = {int(k): int(cont[a]) for a, k in enumerate(ks)}
    return agree, same_ld, same_hd, trust_pen, cont_pen


def _curves_from_counts(agree, m, k_max):
    """metrics.py:208-214."""
    cum = np.cumsum(agree)[1 : k_max + 1]
    k = np.arange(1, k_max + 1)
    q_nx = cum / (k * m)
    r_nx = ((m - 1) * q_nx - k) / (m - 1 - k)
    inv_k = 1.0 / k
    auc = float(np.sum(r_nx * inv_k) / np.sum(inv_k))
    return k, q_nx, r_nx, auc


def _gnn_from_counts(same_ld, same_hd, m, k_max):
    """metrics.py:231-236."""
    k = np.arange(1, k_max + 1)
    g = (np.cumsum(same_ld) - np.cumsum(same_hd)) / (k * m)
    inv_k = 1.0 / k
    auc = float(np.sum(g * inv_k) / np.sum(inv_k))
    return k, g, auc


def rnx_curve(X, Y, k_max=None, device=0):
    """Drop-in for metrics.rnx_curve (metrics.py:185-202): (k, Q_NX, R_NX, AUC)."""
    X, Y = _as_matrix(X), _as_matrix(Y)
    m = X.shape[0]
    if Y.shape[0] != m:
        raise DimensionMismatchError("X and Y row counts differ")
    if m < 4:
        raise InvalidArgumentError("need at least 4 points")
    k_max = default_k_max(m) if k_max is None else int(k_max)
    if not (1 <= k_max <= m - 2):
        raise InvalidArgumentError(f"k_max must be in [1, {m - 2}]")
    agree, _, _, _, _ = _curve_pass(X, Y, None, k_max, (), device=device)
    return _curves_from_counts(agree, m, k_max)


def gnn_curve(X, Y, labels, k_max=None, device=0):
    """Drop-in for metrics.gnn_curve (metrics.py:217-228): (k, G_NN, AUC)."""
    if labels is None:
        raise InvalidArgumentError("kNN gain needs class labels")
    X, Y = _as_matrix(X), _as_matrix(Y)
    m = X.shape[0]
    k_max = default_k_max(m) if k_max is None else int(k_max)
    if not (1 <= k_max <= m - 2):
        raise InvalidArgumentError(f"k_max must be in [1, {m - 2}]")
    _, same_ld, same_hd, _, _ = _curve_pass(X, Y, labels, k_max, (), device=device)
    return _gnn_from_counts(same_ld, same_hd, m, k_max)


def trust_continuity(X, Y, k, device=0):
    """Drop-in for metrics.trust_continuity (metrics.py:240-251)."""
    X, Y = _as_matrix(X), _as_matrix(Y)
    m = X.shape[0]
    if Y.shape[0] != m:
        raise DimensionMismatchError("X and Y row counts differ")
    if not (1 <= k < m / 2):
        raise InvalidArgumentError(f"k must satisfy 1 <= k < M/2, got {k}")
    _, _, _, trust_pen, cont_pen = _curve_pass(X, Y, None, 1, (int(k),), device=device)
    scale = 2.0 / (m * k * (2 * m - 3 * k - 1))
    return 1.0 - scale * trust_pen[int(k)], 1.0 - scale * cont_pen[int(k)]


def evaluate_embedding(X, Y, labels=None, k_max=None, nn_max=100, report_ks=(15, 50, 100), x_precomputed=False,
                       device=0):
    """Drop-in for metrics.evaluate_embedding (metrics.py:351-380): one GPU
    curve pass plus the GPU neighbour hit."""
    Xm = _as_matrix(X)
    Ym = _as_matrix(Y)
    m = Xm.shape[0]
    if Ym.shape[0] != m:
        raise DimensionMismatchError("X and Y row counts differ")
    if m < 4:
        raise InvalidArgumentError("need at least 4 points")
    k_max = default_k_max(m) if k_max is None else min(int(k_max), m - 2)
    report_ks = tuple(int(k) for k in report_ks if k < m / 2)
    lab = None if labels is None else np.asarray(labels)
    agree, same_ld, same_hd, trust_pen, cont_pen = _curve_pass(Xm, Ym, lab, k_max, report_ks,
                                                               x_precomputed=x_precomputed, device=device)
    k, q_nx, r_nx, auc_rnx = _curves_from_counts(agree, m, k_max)
    curves = MetricCurves(k=k, q_nx=q_nx, r_nx=r_nx, auc_rnx=auc_rnx)
    if lab is not None:
        _, g, auc_g = _gnn_from_counts(same_ld, same_hd, m, k_max)
        curves.g_nn, curves.auc_gnn = g, auc_g
        curves.cf_nn, curves.cf = neighbor_hit(Ym, lab, nn_max=min(nn_max, m - 1), device=device)
    for kk in report_ks:
        scale = 2.0 / (m * kk * (2 * m - 3 * kk - 1))
        curves.trust[kk] = 1.0 - scale * trust_pen[kk]
        curves.continuity[kk] = 1.0 - scale * cont_pen[kk]
    return curves


# ------------------------------------------------------ Shepard / co-ranks


def _unrank_pairs(flat, m):
    """Linear upper-triangle index -> (i, j), i < j (reference metrics.py:323-332)."""
    i = (m - 2 - np.floor(np.sqrt(-8.0 * flat + 4.0 * m * (m - 1) - 7) / 2.0 - 0.5)).astype(np.int64)
    j = (flat + i + 1 - (m * (m - 1)) // 2 + ((m - i) * (m - i - 1)) // 2).astype(np.int64)
    return i, j


def _pair_ranks(Z, i_idx, j_idx, device=0):
    """Exact rank of each j among i's neighbours on the GPU (ivhd_pair_ranks;
    reference metrics.py:335-352)."""
    z = np.ascontiguousarray(Z, dtype=np.float64)
    ii = np.ascontiguousarray(i_idx, dtype=np.int64)
    jj = np.ascontiguousarray(j_idx, dtype=np.int64)
    out = np.empty(len(ii), dtype=np.int64)
    lib = _lib.load()
    c_i64 = _lib.ctypes.c_int64
    rc = lib.ivhd_pair_ranks(int(device), _lib.ptr(z, _lib.ctypes.c_double), z.shape[0], int(z.shape[1]),
                             _lib.ptr(ii, c_i64), _lib.ptr(jj, c_i64), len(ii), _lib.ptr(out, c_i64))
    if rc != _lib.OK:
        msg = (lib.ivhd_metrics_last_error() or b"").decode(errors="replace")
        if rc == _lib.ERR_INVALID_ARG:
            raise InvalidArgumentError(msg)
        raise DeviceError(f"pair ranks failed: {msg}")
    return out


def shepard_and_corank(X, Y, sample_pairs=10000, seed=0, device=0):
    """Drop-in for metrics.shepard_and_corank (metrics.py:297-320): sampled
    distance pairs, their exact ranks in X and Y (GPU), and R^2 of the
    co-ranks against the identity.  Pair sampling is the reference's."""
    X, Y = _as_matrix(X), _as_matrix(Y)
    m = X.shape[0]
    if Y.shape[0] != m:
        raise DimensionMismatchError("X and Y row counts differ")
    total = m * (m - 1) // 2
    if sample_pairs > total:
        raise InvalidArgumentError(f"at most {total} distinct pairs exist")
    rng = np.random.default_rng(seed)
    flat = rng.choice(total, size=sample_pairs, replace=False)
    i_idx, j_idx = _unrank_pairs(flat, m)
    deltas = np.linalg.norm(X[i_idx] - X[j_idx], axis=1)
    dists = np.linalg.norm(Y[i_idx] - Y[j_idx], axis=1)
    rho = _pair_ranks(X, i_idx, j_idx, device=device)
    r = _pair_ranks(Y, i_idx, j_idx, device=device)
    resid = r.astype(np.float64) - rho.astype(np.float64)
    centered = r - r.mean()
    ss_tot = float(np.sum(centered * centered))
    r2 = 1.0 - float(np.sum(resid * resid)) / ss_tot if ss_tot > 0 else 1.0
    return (deltas, dists), (rho, r), r2


# ----------------------------------------------------------- rank matrices


@dataclass
class RankData:
    """Full rank matrices for a (X, Y) pair; rank[i, i] is 0 (metrics.py:18-23)."""

    hd_ranks: np.ndarray
    ld_ranks: np.ndarray | None = None


def _rank_matrix(source, precomputed, device=0):
    src = np.ascontiguousarray(source, dtype=np.float64)
    m = src.shape[0]
    out = np.empty((m, m), dtype=np.int64)
    lib = _lib.load()
    rc = lib.ivhd_rank_matrix(int(device), _lib.ptr(src, _lib.ctypes.c_double), m, int(src.shape[1]),
                              int(bool(precomputed)), _lib.ptr(out, _lib.ctypes.c_int64))
    if rc != _lib.OK:
        msg = (lib.ivhd_metrics_last_error() or b"").decode(errors="replace")
        if rc == _lib.ERR_INVALID_ARG:
            raise InvalidArgumentError(msg)
        raise DeviceError(f"rank matrix failed: {msg}")
    return out


def compute_ranks(distances=None, dataset=None, ld_distances=None, device=0):
    """Drop-in for metrics.compute_ranks (metrics.py:116-146): exact rank
    matrices under the index tie rule, computed on the GPU (ivhd_rank_matrix)."""
    if (distances is None) == (dataset is None):
        raise InvalidArgumentError("pass exactly one of distances / dataset")
    if distances is not None:
        D = _as_matrix(distances)
        if D.shape[0] != D.shape[1]:
            raise DimensionMismatchError("distance matrix must be square")
        source, pre = D, True
    else:
        source, pre = _as_matrix(dataset), False
    if source.shape[0] < 2:
        raise InvalidArgumentError("need at least two points to rank")
    hd = _rank_matrix(source, pre, device=device)
    ld = None
    if ld_distances is not None:
        ld = compute_ranks(distances=ld_distances, device=device).hd_ranks
    return RankData(hd_ranks=hd, ld_ranks=ld)
