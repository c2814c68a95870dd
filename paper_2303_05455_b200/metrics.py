"""Embedding quality metrics on the GPU.

`neighbor_hit` is the drop-in for the reference's `ivhd.metrics.neighbor_hit`
(/root/reference/pkg/src/ivhd/metrics.py:254-294): same signature, same
(cf_nn, cf) result.  For embedded points the nn_max nearest neighbours come
from the exact grid kNN in csrc/ivhd_metrics.cu (2-D/3-D); for a prebuilt
KnnGraph the reference's arithmetic on the given neighbour block is applied
directly (label comparisons only, no search).
"""

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
