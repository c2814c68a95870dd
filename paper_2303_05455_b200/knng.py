"""Exact kNN graph construction on the GPU — the drop-in for the reference's
`ivhd.knng.build_exact_knn` (/root/reference/pkg/src/ivhd/knng.py:158-194).

Same signature and result: a `KnnGraph` whose row i lists the k nearest other
rows of the input ordered by (distance, index), with float64 distances.  The
work runs in libivhd_b200.so (csrc/ivhd_knn.cu): a tcgen05 tensor-core
candidate pass, an exact fp64 re-rank with an error-bounded certificate, and
an exact fp64 scan for any row the certificate does not cover.  There is no
CPU path.

Metrics: "euclidean" and "cosine" (knng.py:105-115, 185-189) through the
tensor-core pass; "precomputed" (a square distance matrix, knng.py:175-181)
through a warp-per-row streaming top-k (k <= 128).
"""

import os
import time

import numpy as np

from . import _lib
from .embed import KnnGraph
from .errors import DegenerateMetricError, DeviceError, DimensionMismatchError, InvalidArgumentError

_METRICS = {"euclidean": 0, "cosine": 1, "precomputed": 2}

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
    if metric == "precomputed" and (data.ndim != 2 or data.shape[0] != data.shape[1]):
        raise DimensionMismatchError("precomputed metric needs a square matrix")
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


# ------------------------------------------------------------- graph cache
# The reference's binary cache (knng.py:286-332): b"IVHG", then <u4
# [version=1, M, k, metric id, has_dist], the (M, k) <u4 neighbour block and,
# if flagged, the (M, k) <f4 distance block.

_CACHE_MAGIC = b"IVHG"
_METRIC_IDS = {"euclidean": 0, "cosine": 1, "precomputed": 2}


def cache_write(graph, path):
    """Write `graph` in the reference's IVHG format (knng.py:286-300):
    byte-identical to the reference writer — its header layout and field
    order are the reference's, kept as is so either side reads the other's
    files."""
    from .errors import MalformedInputError

    has_dist = graph.distances is not None
    metric = getattr(graph, "metric", "euclidean")
    header = np.asarray([1, graph.neighbors.shape[0], graph.neighbors.shape[1], _METRIC_IDS[metric],
                         int(has_dist)], dtype="<u4")
    try:
        with open(path, "wb") as fh:
            fh.write(_CACHE_MAGIC)
            fh.write(header.tobytes())
            fh.write(np.ascontiguousarray(graph.neighbors, dtype="<u4").tobytes())
            if has_dist:
                fh.write(np.ascontiguousarray(graph.distances, dtype="<f4").tobytes())
    except OSError as exc:
        raise MalformedInputError(f"{path}: cannot write graph cache: {exc}")


def cache_read(path, distances=True):
    """Read an IVHG cache (knng.py:303-332).  The neighbour block is
    memory-mapped, not copied: `run_embedding` hands the mapping straight to
    the device CSR builder (ivhd_set_graph reads it once, H2D), so a 10^8-row
    graph is never duplicated in host memory.  Same errors as the reference
    (MalformedInputError on a bad magic, version or a truncated file)."""
    from .errors import MalformedInputError

    try:
        with open(path, "rb") as fh:
            head = fh.read(24)
        size = os.path.getsize(path)
    except OSError as exc:
        raise MalformedInputError(f"{path}: cannot read graph cache: {exc}")
    if head[:4] != _CACHE_MAGIC:
        raise MalformedInputError(f"{path}: not a graph cache file")
    if len(head) < 24:
        raise MalformedInputError(f"{path}: truncated graph cache")
    version, m, k, metric_id, has_dist = np.frombuffer(head[4:24], dtype="<u4")
    if version != 1:
        raise MalformedInputError(f"{path}: unsupported cache version {version}")
    nbytes = int(m) * int(k) * 4
    if size < 24 + nbytes * (1 + int(has_dist)):
        raise MalformedInputError(f"{path}: truncated graph cache")
    # ids < 2^31, so the <u4 block reads as int32 without conversion
    nbr = np.memmap(path, dtype="<i4", mode="r", offset=24, shape=(int(m), int(k))) if nbytes else \
        np.empty((int(m), int(k)), dtype=np.int32)
    dist = None
    if has_dist and distances and nbytes:
        dist = np.memmap(path, dtype="<f4", mode="r", offset=24 + nbytes, shape=(int(m), int(k))).astype(np.float64)
    metric = {v: key for key, v in _METRIC_IDS.items()}[int(metric_id)]
    return KnnGraph(nbr, dist, metric=metric)
