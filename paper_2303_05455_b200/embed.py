"""`run_embedding` — the drop-in entry point (reference engine.py:312-414).

Same signature, same return type shape (RunResult(embedding, trace, state,
mutations)), same exceptions, same RNG stream.  What moved: the loop body.
The reference evaluates forces with numpy gathers and bincounts and updates
positions on the CPU once per iteration; here the whole particle system lives
on the GPU and `DeviceEmbedding.run` executes whole phase segments as CUDA
graph replays of one fused kernel per iteration (ivhd_step.cuh).  The host
only (a) replays the seeded setup draws that must be bit-identical to the
reference (initial layout, random neighbours, resampling), (b) splits the
run into segments at phase boundaries / resampling points, and (c) talks to
an observer between iterations when one is attached.
"""

import sys
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .config import EmbeddingConfig, coerce_config, resolve_optimizer
from .config import OPTIMIZER_KINDS
from .device import DeviceEmbedding, is_pcg64
from .errors import (DimensionMismatchError, InvalidArgumentError,
                     NumericalDivergenceError)


# ------------------------------------------------------------------- types


@dataclass
class Embedding:
    """Output points (M x 2 or 3, float64) + optional labels (datasets.py:80-100)."""

    points: np.ndarray
    labels: np.ndarray | None = None

    def __post_init__(self):
        self.points = np.asarray(self.points, dtype=np.float64)
        if self.points.ndim != 2 or self.points.shape[1] not in (2, 3):
            raise DimensionMismatchError(
                f"embedding must be M x 2 or M x 3, got shape {self.points.shape}")

    @property
    def M(self):
        return self.points.shape[0]


@dataclass
class KnnGraph:
    """Minimal input container (knng.py:27-69): neighbors (M,k) int32,
    optional distances (M,k).  The reference's KnnGraph works as well."""

    neighbors: np.ndarray
    distances: np.ndarray | None = None
    metric: str = "euclidean"

    def __post_init__(self):
        self.neighbors = np.asarray(self.neighbors, dtype=np.int32)
        if self.neighbors.ndim != 2:
            raise DimensionMismatchError("neighbors must be an M x k matrix")
        if self.distances is not None:
            self.distances = np.asarray(self.distances, dtype=np.float64)
            if self.distances.shape != self.neighbors.shape:
                raise DimensionMismatchError("distances shape must match neighbors")

    @property
    def M(self):
        return self.neighbors.shape[0]

    @property
    def k(self):
        return self.neighbors.shape[1]


@dataclass
class EmbeddingState:
    """engine.py:87-95."""

    positions: np.ndarray
    deltas: np.ndarray
    rn_assignments: np.ndarray
    iteration: int = 0
    stress: float = float("nan")


@dataclass
class StressTrace:
    """engine.py:98-113."""

    iterations: list = field(default_factory=list)
    stress: list = field(default_factory=list)
    step_size: list = field(default_factory=list)

    def append(self, iteration, stress, step_size):
        self.iterations.append(int(iteration))
        self.stress.append(float(stress))
        self.step_size.append(float(step_size))

    def extend(self, first, stress, step):
        n = len(stress)
        self.iterations.extend(range(int(first), int(first) + n))
        self.stress.extend(float(s) for s in stress)
        self.step_size.extend(float(b) for b in step)

    def to_csv(self, path):
        rows = ["iteration,stress,b"]
        rows += [f"{i},{s!r},{b!r}" for i, s, b in zip(self.iterations, self.stress, self.step_size)]
        with open(path, "w") as fh:
            fh.write("\n".join(rows) + "\n")


@dataclass
class RunResult:
    """engine.py:116-121."""

    embedding: Embedding
    trace: StressTrace
    state: EmbeddingState
    mutations: list = field(default_factory=list)


# ----------------------------------------------------- seeded setup draws


def init_layout(m, target_dim, seed):
    """Uniform positions in [-1, 1]^dim (engine.py:124-129); bit-identical
    to the reference for the same generator state."""
    if m < 1:
        raise InvalidArgumentError("need at least one point")
    gen = seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)
    return gen.uniform(-1.0, 1.0, size=(m, target_dim))


def sample_random_neighbors(m, nn_sets, rn, seed):
    """Random partners, uniform over ids that are neither self nor an nn
    (engine.py:132-146).  Rejected slots are re-drawn in row-major order, which
    keeps the PCG64 stream identical to the reference."""
    nn_sets = np.asarray(nn_sets)
    if m <= nn_sets.shape[1] + rn:
        raise InvalidArgumentError(f"M={m} too small for nn={nn_sets.shape[1]} plus rn={rn}")
    gen = seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)
    picks = gen.integers(0, m, size=(m, rn))
    ids = np.arange(m)[:, None]
    while True:
        reject = picks == ids
        for col in range(nn_sets.shape[1]):
            reject |= picks == nn_sets[:, col : col + 1]
        n_reject = int(np.count_nonzero(reject))
        if n_reject == 0:
            return picks.astype(np.int32)
        picks[reject] = gen.integers(0, m, size=n_reject)


def rnn_edge_filter(nn_edges, nn_sets, helper_graph):
    """Keep nn pair (i, j) iff i is in helper-kNN(j); a point whose every pair
    fails keeps column 0 (engine.py:289-309)."""
    nb = np.asarray(getattr(helper_graph, "neighbors", helper_graph))
    claims = nb[nn_edges[:, 1]] == nn_edges[:, 0][:, None]
    keep = claims.any(axis=1)
    m, ncols = nn_sets.shape
    rows = keep.reshape(m, ncols)
    empty = ~rows.any(axis=1)
    if empty.any():
        rows = rows.copy()
        rows[empty, 0] = True
        keep = rows.reshape(-1)
    return keep


def _pair_distances(data, src, dst, metric):
    """Feature-space distance of random pairs (knng.py:197-204)."""
    a, b = data[src], data[dst]
    if metric == "cosine":
        return np.maximum(1.0 - np.einsum("ij,ij->i", a, b), 0.0)
    d = a - b
    return np.sqrt(np.einsum("ij,ij->i", d, d))


def _phase_name(rnn_on, l1_on):
    return {(True, True): "rnn+l1", (True, False): "rnn", (False, True): "l1"}.get(
        (rnn_on, l1_on), "main")


# ------------------------------------------------------------------ session


class _Session:
    """Setup of one run (engine.py:162-221) with the particle system on the GPU."""

    def __init__(self, graph, config, dataset, helper_graph, device, make_device=None):
        self.config = config
        self.rng = np.random.default_rng(config.seed)
        self.data = None if dataset is None else np.asarray(dataset.data, dtype=np.float64)
        self.labels = None if dataset is None else getattr(dataset, "labels", None)
        if graph is None:
            if dataset is None:
                raise InvalidArgumentError("need a graph or a dataset to embed")
            # engine.py:170-176: the exact kNN graph of the dataset (GPU builder)
            from .knng import build_exact_knn

            k = config.nn * 4 if config.rnn_final_steps > 0 else config.nn
            graph = build_exact_knn(dataset, min(k, self.data.shape[0] - 1), config.graph_metric,
                                    device=device)
        self.graph = graph
        neighbors = np.asarray(graph.neighbors)
        m, k = neighbors.shape
        self.m = m
        ncols = min(config.nn, k)
        if k < config.nn:
            warnings.warn(f"graph stores k={k} < nn={config.nn}; using all stored neighbors",
                          stacklevel=3)
        self.nn_sets = neighbors[:, :ncols]

        self.helper = None
        if config.rnn_final_steps > 0:
            if helper_graph is not None:
                self.helper = helper_graph
            elif k >= min(4 * config.nn, m - 1):
                self.helper = graph
            elif self.data is not None:  # engine.py:194-199
                from .knng import build_exact_knn

                self.helper = build_exact_knn(dataset, min(4 * config.nn, m - 1), config.graph_metric,
                                              device=device)
            else:
                raise InvalidArgumentError(
                    "reverse-neighbor phase needs a helper graph or the dataset")

        self.euclid = config.distance_mode == "euclidean"
        if self.euclid:
            if getattr(graph, "distances", None) is None:
                raise InvalidArgumentError("euclidean mode needs stored graph distances")
            if self.data is None:
                raise InvalidArgumentError(
                    "euclidean mode needs the dataset to measure random-pair targets")

        self.c = config.c
        self.target_scale = None
        self.dim = config.target_dim
        if m <= self.nn_sets.shape[1] + config.rn:
            raise InvalidArgumentError(f"M={m} too small for nn={self.nn_sets.shape[1]} plus rn={config.rn}")

        # one GPU (DeviceEmbedding) or this rank's shard (sharded.ShardedEmbedding)
        self.dev = (make_device or DeviceEmbedding)(m, config.target_dim, device=device)
        # degenerate random pairs draw their directions from this run's
        # generator on the host (degenerate.py, forces.py:167-174)
        getattr(self.dev, "device_embedding", self.dev).degenerate_resolver = self.degenerate_directions
        self.dev.set_optimizer(resolve_optimizer(config.optimizer, m, config.integrator, config.opt))
        # one PCG64 stream, reference order (engine.py:165, 214-215): the
        # layout, then the random partners — drawn on the device (numpy's
        # PCG64 reproduced bit for bit; the host Generator is advanced to match)
        self.device_rng = is_pcg64(self.rng)
        self._y0 = None
        if self.device_rng:
            self._y0_state = self.rng.bit_generator.state
            self.dev.init_positions(self.rng)
        else:
            self._y0 = init_layout(m, config.target_dim, self.rng)
            self.dev.set_positions(self._y0)
        self.rn = None
        self._upload_connections(sample=True)

    @property
    def y0(self):
        """The initial layout (host copy, replayed from the saved generator
        state when the device drew it)."""
        if self._y0 is None:
            g = np.random.Generator(np.random.PCG64())
            g.bit_generator.state = self._y0_state
            self._y0 = init_layout(self.m, self.dim, g)
        return self._y0

    # connection sets ------------------------------------------------------
    def _targets(self):
        """Euclidean targets (engine.py:229-253), scaled once by 1/max."""
        ncols = self.nn_sets.shape[1]
        nn_t = np.asarray(self.graph.distances)[:, :ncols].reshape(-1).astype(np.float64)
        src = np.repeat(np.arange(self.m), self.rn.shape[1])
        rn_t = _pair_distances(self.data, src, self.rn.reshape(-1),
                               getattr(self.graph, "metric", "euclidean"))
        if self.config.normalize_targets:
            if self.target_scale is None:
                peak = max(float(nn_t.max(initial=0.0)), float(rn_t.max(initial=0.0)))
                self.target_scale = 1.0 / peak if peak > 0 else 1.0
            nn_t = nn_t * self.target_scale
            rn_t = rn_t * self.target_scale
        return nn_t, rn_t

    def _edge_arrays(self):
        m, ncols = self.nn_sets.shape
        rn = self.rn.shape[1]
        nn_edges = np.column_stack([np.repeat(np.arange(m, dtype=np.int32), ncols),
                                    self.nn_sets.reshape(-1).astype(np.int32)])
        rn_edges = np.column_stack([np.repeat(np.arange(m, dtype=np.int32), rn),
                                    self.rn.reshape(-1).astype(np.int32)])
        return nn_edges, rn_edges

    def _upload_connections(self, sample=False):
        self.filtered_ready = False
        if not self.euclid:
            if sample and self.device_rng:
                self.rn = self.dev.set_graph_sampled(0, self.nn_sets, self.config.rn, self.rng)
                return
            if sample:
                self.rn = sample_random_neighbors(self.m, self.nn_sets, self.config.rn, self.rng)
            self.dev.set_graph(0, self.nn_sets, self.rn)
            return
        if sample:
            self.rn = sample_random_neighbors(self.m, self.nn_sets, self.config.rn, self.rng)
        nn_t, rn_t = self._targets()
        nn_edges, rn_edges = self._edge_arrays()
        self.dev.set_connections(
            0, np.vstack([nn_edges, rn_edges]),
            np.repeat([0, 1], [len(nn_edges), len(rn_edges)]).astype(np.uint8),
            np.concatenate([nn_t, rn_t]))

    def ensure_filtered(self):
        """Slot 1 = RNN-filtered set with per-edge budget scale (engine.py:270-286)."""
        if self.filtered_ready:
            return
        nn_edges, rn_edges = self._edge_arrays()
        if self.euclid:
            nn_t, rn_t = self._targets()
        else:
            nn_t, rn_t = np.zeros(len(nn_edges)), np.ones(len(rn_edges))
        keep = rnn_edge_filter(nn_edges, self.nn_sets, self.helper)
        ncols = self.nn_sets.shape[1]
        kept_per = keep.reshape(-1, ncols).sum(axis=1)
        scale = (ncols / kept_per)[nn_edges[keep][:, 0]]
        n_keep = int(keep.sum())
        self.dev.set_connections(
            1, np.vstack([nn_edges[keep], rn_edges]),
            np.repeat([0, 1], [n_keep, len(rn_edges)]).astype(np.uint8),
            np.concatenate([nn_t[keep], rn_t]),
            np.concatenate([scale, np.ones(len(rn_edges))]))
        self.filtered_ready = True

    def connection_arrays(self, slot):
        """(src, dst, w * t) of connection set `slot` in the reference's
        connection order (engine.py:225-262; slot 1 = rnn_filtered, 270-286)."""
        nn_edges, rn_edges = self._edge_arrays()
        if self.euclid:
            nn_t, rn_t = self._targets()
        else:
            nn_t, rn_t = np.zeros(len(nn_edges)), np.ones(len(rn_edges))
        nn_w = np.ones(len(nn_edges))
        if slot == 1:
            keep = rnn_edge_filter(nn_edges, self.nn_sets, self.helper)
            ncols = self.nn_sets.shape[1]
            kept_per = keep.reshape(-1, ncols).sum(axis=1)
            nn_edges, nn_t = nn_edges[keep], nn_t[keep]
            nn_w = (ncols / kept_per)[nn_edges[:, 0]]
        src = np.concatenate([nn_edges[:, 0], rn_edges[:, 0]])
        dst = np.concatenate([nn_edges[:, 1], rn_edges[:, 1]])
        wt = np.concatenate([nn_w * nn_t, self.c * rn_t])
        return src, dst, wt

    def degenerate_directions(self, slot, rows, entries):
        from . import degenerate

        src, dst, wt = self.connection_arrays(slot)
        return degenerate.table(rows, entries, src, dst, wt, self.rng, self.dim)

    def resample(self):
        """engine.py:264-268: new random partners from the same stream."""
        self._upload_connections(sample=True)

    def set_optimizer(self, kind):
        self.config.optimizer = kind
        self.dev.set_optimizer(resolve_optimizer(kind, self.m, self.config.integrator,
                                                 self.config.opt))


def _apply_mutation(sess, key, value):
    """engine.py:417-448; returns the applied value (or raises)."""
    if key == "c":
        value = float(value)
        if not 0.0 < value < 1.0:
            raise InvalidArgumentError(f"c must be in (0, 1), got {value}")
        sess.c = value
        return value
    if key == "b":
        value = float(value)
        if value <= 0:
            raise InvalidArgumentError(f"step size must be positive, got {value}")
        # ForceDirected.params.b / Sgd..Adam .alpha; Adadelta has neither
        # attribute, so the reference leaves its scale untouched (engine.py:428-431)
        if sess.config.optimizer != "adadelta":
            sess.dev.set_step_size(value)
        return value
    if key == "optimizer":
        if value not in OPTIMIZER_KINDS:
            raise InvalidArgumentError(f"unknown optimizer {value!r}")
        sess.set_optimizer(value)
        return value
    if key == "rn_resample_period":
        value = int(value)
        if value < 0:
            raise InvalidArgumentError("rn_resample_period must be >= 0")
        return value
    if key in ("start_l1", "start_rnn", "stop"):
        return bool(value)
    raise InvalidArgumentError(f"unknown mutation {key!r}")


# --------------------------------------------------------------- the loop


class LazyPositions:
    """Positions handed to an observer (steering fast
    path): the device → host copy happens only when the observer reads them
    (np.asarray, indexing, len, .copy(), any ndarray attribute), so an
    observer that publishes a frame every N iterations (server.py:103-116)
    pays the (M, dim) transfer once per frame, not once per iteration.  If the
    observer keeps a reference past its return, the loop materialises the
    object before the next iteration, so it always holds that iteration's
    positions."""

    __slots__ = ("_dev", "_arr", "shape")

    def __init__(self, dev, m, dim):
        self._dev = dev
        self._arr = None
        self.shape = (m, dim)

    def _get(self):
        if self._arr is None:
            self._arr = self._dev.positions()
            self._dev = None
        return self._arr

    materialize = _get

    def __array__(self, dtype=None, copy=None):
        a = self._get()
        if dtype is not None and a.dtype != dtype:
            return a.astype(dtype)
        return a.copy() if copy else a

    def __len__(self):
        return self.shape[0]

    def __getitem__(self, key):
        return self._get()[key]

    def __iter__(self):
        return iter(self._get())

    def __getattr__(self, name):  # ndarray API (copy, mean, min, tolist, ...)
        return getattr(self._get(), name)

    def __repr__(self):
        return repr(self._get())


def run_embedding(graph=None, config=None, dataset=None, helper_graph=None, observer=None,
                  threads=1, device=0):
    """Execute a full embedding run on the GPU (engine.py:312-414).

    observer(iteration, positions, stress, params) is called between
    iterations and may return mutations {"c", "b", "optimizer",
    "rn_resample_period", "start_l1", "start_rnn", "stop"}.  `threads` is
    accepted for signature compatibility (the reference's phase-1 pool size)
    and ignored.  Raises NumericalDivergenceError with the last finite state.
    """
    del threads
    config = coerce_config(config)
    sess = _Session(graph, config, dataset, helper_graph, device)
    return _drive(sess, config, observer)


def _drive(sess, config, observer):
    """The loop of engine.py:331-414 over device segments (shared by
    run_embedding and sharded.run_embedding_distributed)."""
    dev = sess.dev
    total = config.iterations
    trace = StressTrace()
    mutations = []
    l1_from = total - config.l1_final_steps if config.l1_final_steps > 0 else None
    rnn_from = total - config.rnn_final_steps if config.rnn_final_steps > 0 else None
    period = config.rn_resample_period
    state = EmbeddingState(positions=None, deltas=None, rn_assignments=sess.rn, iteration=0)

    def diverged(it0, stress, done):
        state.positions = dev.positions()
        state.iteration = it0 + done
        state.stress = float(stress[done])
        state.deltas = dev.deltas()
        state.rn_assignments = sess.rn
        raise NumericalDivergenceError(it0 + done, state)

    ran = 0
    it = 0
    stop = False
    while it < total and not stop:
        if period > 0 and it > 0 and it % period == 0:
            sess.resample()
            state.rn_assignments = sess.rn
        rnn_on = rnn_from is not None and it >= rnn_from
        l1_on = l1_from is not None and it >= l1_from
        if rnn_on and sess.helper is None:
            raise InvalidArgumentError("reverse-neighbor phase needs a helper graph or the dataset")
        slot = 0
        if rnn_on:
            sess.ensure_filtered()
            slot = 1
        norm = "l1" if l1_on else "l2"
        if observer is None:
            # one device segment up to the next phase switch / resample point
            end = total
            for edge in (rnn_from, l1_from):
                if edge is not None and it < edge < end:
                    end = edge
            if period > 0:
                end = min(end, (it // period + 1) * period)
        else:
            end = it + 1
        stress, step, done, div = dev.run(slot, norm, sess.c, end - it)
        trace.extend(it, stress[:done], step[:done])
        if div:
            diverged(it, stress, done)
        ran += done
        if observer is not None:
            positions = LazyPositions(dev, sess.m, sess.dim)
            energy = float(stress[0])
            state.positions = positions
            state.iteration = it + 1
            state.stress = energy
            snapshot = {"c": sess.c, "b": float(step[0]), "optimizer": config.optimizer,
                        "phase": _phase_name(rnn_on, l1_on)}
            requested = observer(it, positions, energy, snapshot)
            if sys.getrefcount(positions) > 3:  # kept by the observer (or state): pin this iteration's values
                positions.materialize()
            for key, value in (requested or {}).items():
                applied = _apply_mutation(sess, key, value)
                if applied is not None:
                    mutations.append((it, key, applied))
                if key == "stop":
                    stop = True
                elif key == "start_l1":
                    l1_from = it + 1
                elif key == "start_rnn":
                    rnn_from = it + 1
                elif key == "rn_resample_period":
                    period = int(value)
        else:
            state.iteration = end
            state.stress = float(stress[done - 1])
        it = end

    # result arrays in recycled page-locked host memory (_lib.PinnedPool): the
    # copies run at link rate with no first-touch faults; the embedding gets its
    # own copy of the final positions (engine.py:413), read from the device again
    shape = (sess.m, sess.dim)
    positions = dev.positions(out=_lib.pinned.empty(shape, dev.device)) if ran else sess.y0.copy()
    state.positions = positions
    state.rn_assignments = sess.rn
    state.deltas = dev.deltas(out=_lib.pinned.empty(shape, dev.device)) if ran else np.zeros(shape)
    if total == 0 or state.stress != state.stress:
        state.stress = dev.stress(0, "l2", sess.c, positions)
    emb_points = dev.positions(out=_lib.pinned.empty(shape, dev.device)) if ran else positions.copy()
    dev.close()
    emb = Embedding(emb_points, labels=sess.labels)
    return RunResult(embedding=emb, trace=trace, state=state, mutations=mutations)
