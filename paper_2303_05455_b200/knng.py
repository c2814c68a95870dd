"""Exact kNN graph construction on the GPU — the drop-in for the reference's
`ivhd.knng.build_exact_knn` (/root/reference/pkg/src/ivhd/knng.py:158-194).

Same signature and result: a `KnnGraph` whose row i lists the k nearest other
rows of the input ordered by (distance, index), with float64 distances.  The
work runs in libivhd_b200.so (csrc/ivhd_knn.cu): a tcgen05 tensor-core
candidate pass, an exact fp64 re-rank with an error-bounded certificate, and
an exact fp64 scan for any row the certificate does not cover.  There is no
CPU path.

Metrics: "euclidean" and "cosine" (knng.py:105-115, 185-189).  "precomputed"
(a square distance matrix) is not a GPU path here and raises
InvalidArgumentError.
"""

import time

import numpy as np

from . import _lib
from .embed import KnnGraph
from .errors import DegenerateMetricError, DeviceError, DimensionMismatchError, InvalidArgumentError

_METRICS = {"euclidean": 0, "cosine": 1}

last_stats = {}


def build_exact_knn(dataset_or_matrix, k, metric="euclidean", chunk_budget=None, device=0):
    """Exact kNN graph (knng.py:158-194); `chunk_budget` is accepted for
    signature compatibility and ignored (the GPU kernel streams tiles)."""
    data = getattr(dataset_or_matrix, "data", dataset_or_matrix)
    data = np.asarray(data)
    if data.ndim != 2:
        raise DimensionMismatchError("kNN input must be an (M, N) matrix")
    m = data.shape[0]
    k = int(k)
    if not (1 <= k < m):
        raise InvalidArgumentError(f"k must satisfy 1 <= k < M, got k={k}, M={m}")
    if metric == "precomputed":
        raise InvalidArgumentError("precomputed metric is not supported by the GPU kNN builder")
    if metric not in _METRICS:
        raise InvalidArgumentError(f"unknown metric {metric!r}")
    x = _lib.f64(data)
    lib = _lib.load()
    nbr = np.empty((m, k), dtype=np.int32)
    dist = np.empty((m, k), dtype=np.float64)
    stats = np.zeros(8, dtype=np.float64)
    t0 = time.perf_counter()
    rc = lib.ivhd_knn_build(int(device), _lib.ptr(x, _lib.ctypes.c_double), m, int(x.shape[1]), k,
                            _METRICS[metric], _lib.ptr(nbr, _lib.ctypes.c_int32),
                            _lib.ptr(dist, _lib.ctypes.c_double), _lib.ptr(stats, _lib.ctypes.c_double))
    if rc != _lib.OK:
        msg = (lib.ivhd_knn_last_error() or b"").decode(errors="replace")
        if rc == _lib.ERR_INVALID_ARG and "zero-norm" in msg:
            row = int(msg.rsplit("row", 1)[1].strip(" )")) if "row" in msg else None
            raise DegenerateMetricError("zero-norm vector under cosine metric", row=row)
        if rc == _lib.ERR_INVALID_ARG:
            raise InvalidArgumentError(msg)
        raise DeviceError(f"kNN build failed: {msg}")
    last_stats.clear()
    last_stats.update(tc_seconds=stats[0], rerank_seconds=stats[1], exact_rows=int(stats[2]),
                      device_seconds=stats[3], setup_seconds=stats[4], exact_seconds=stats[5],
                      d2h_seconds=stats[6], wall_seconds=time.perf_counter() - t0)
    return KnnGraph(nbr, dist, metric=metric)
