"""B200-native IVHD embedding loop (arXiv 2303.05455), drop-in for the
reference package's `run_embedding` hot path.

Host code here is Python; the loop runs in libivhd_b200.so (hand-written
sm_100a CUDA behind the C ABI in include/ivhd_b200.h).
"""

from .config import (DEFAULT_ALPHA, OPTIMIZER_KINDS, EmbeddingConfig, IntegratorParams,
                     OptimizerParams)
from .embed import (Embedding, EmbeddingState, KnnGraph, RunResult, StressTrace,
                    init_layout, rnn_edge_filter, run_embedding, sample_random_neighbors)
from .errors import (DeviceError, DimensionMismatchError, InvalidArgumentError, IvhdError,
                     NumericalDivergenceError)
from .operators import ConnectionSet, compute_forces, gradient, stress

__version__ = "0.1.0"

__all__ = [
    "ConnectionSet", "DEFAULT_ALPHA", "DeviceError", "DimensionMismatchError", "Embedding",
    "EmbeddingConfig", "EmbeddingState", "IntegratorParams", "InvalidArgumentError",
    "IvhdError", "KnnGraph", "NumericalDivergenceError", "OPTIMIZER_KINDS", "OptimizerParams",
    "RunResult", "StressTrace", "compute_forces", "gradient", "init_layout", "rnn_edge_filter",
    "run_embedding", "sample_random_neighbors", "stress",
]
