"""Thin owner of one `ivhd_ctx` (include/ivhd_b200.h).

`DeviceEmbedding` keeps the whole particle system resident on one GPU: the
symmetrised CSR of the main and the RNN-filtered connection sets, the two
position buffers, the optimizer state and the trace.  Every method is a
synchronous C-ABI call; nothing here computes on the CPU.
"""

import ctypes

import numpy as np

from . import _lib
from ._lib import c_f64p, c_i32p, c_i64p, c_u8p, c_u64p, check, f64, i32, ptr
from .errors import InvalidArgumentError


_M64 = (1 << 64) - 1


def is_pcg64(gen):
    return type(getattr(gen, "bit_generator", None)).__name__ == "PCG64"


def pcg_state(gen):
    """numpy PCG64 state as the C ABI's rng[6] words."""
    if not is_pcg64(gen):
        raise InvalidArgumentError("device draws need a numpy Generator backed by PCG64")
    st = gen.bit_generator.state
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    return np.array([s >> 64, s & _M64, inc >> 64, inc & _M64, int(st["has_uint32"]), int(st["uinteger"])],
                    dtype=np.uint64)


def pcg_store(gen, words):
    st = gen.bit_generator.state
    st["state"]["state"] = (int(words[0]) << 64) | int(words[1])
    st["state"]["inc"] = (int(words[2]) << 64) | int(words[3])
    st["has_uint32"] = int(words[4])
    st["uinteger"] = int(words[5])
    gen.bit_generator.state = st


class DeviceEmbedding:
    def __init__(self, m, dim, device=0, stream=0):
        self.lib = _lib.load()
        self.m = int(m)
        self.dim = int(dim)
        self.device = int(device)
        h = ctypes.c_void_p()
        check(self.lib.ivhd_create(ctypes.byref(h), int(device), self.m, self.dim, int(stream)))
        self.h = h

    # ------------------------------------------------------------ lifetime
    def close(self):
        if getattr(self, "h", None):
            self.lib.ivhd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, code):
        check(code, self.h)

    # ---------------------------------------------------------- connections
    def _nn_view(self, nn_sets):
        nn = np.asarray(nn_sets)
        if nn.ndim != 2 or nn.shape[0] != self.m:
            raise InvalidArgumentError("nn_sets must be (M, ncols)")
        base = nn if (nn.dtype == np.int32 and nn.strides[1] == 4) else i32(nn)
        stride = base.strides[0] // 4 if base.shape[1] > 0 else 0
        if base.strides[0] % 4 or stride < base.shape[1]:
            base = i32(nn)
            stride = base.shape[1]
        return base, stride

    def set_graph(self, slot, nn_sets, rn_assign):
        """Binary-mode connections: nn (M, ncols) view (row stride honoured)
        and rn (M, rn).  engine.py:225-262."""
        base, stride = self._nn_view(nn_sets)
        rn = i32(rn_assign)
        self._check(self.lib.ivhd_set_graph(
            self.h, int(slot), base.ctypes.data_as(c_i32p) if base.size else None, int(stride),
            int(base.shape[1]), rn.ctypes.data_as(c_i32p) if rn.size else None,
            int(rn.shape[1]) if rn.ndim == 2 else 0))

    def set_graph_sampled(self, slot, nn_sets, rn, gen):
        """Draw rn random partners per vertex on the device from the numpy
        Generator `gen` (PCG64) exactly as sample_random_neighbors would
        (engine.py:132-146), advance `gen` accordingly, and build the binary
        connection set.  Returns the (M, rn) int32 partners."""
        base, stride = self._nn_view(nn_sets)
        st = pcg_state(gen)
        picks = np.empty((self.m, int(rn)), dtype=np.int32)
        self._check(self.lib.ivhd_set_graph_sampled(
            self.h, int(slot), base.ctypes.data_as(c_i32p) if base.size else None, int(stride),
            int(base.shape[1]), int(rn), st.ctypes.data_as(c_u64p),
            picks.ctypes.data_as(c_i32p) if picks.size else None))
        pcg_store(gen, st)
        return picks

    def init_positions(self, gen, low=-1.0, high=1.0):
        """positions = gen.uniform(low, high, (M, dim)) drawn on the device
        (engine.py:124-129); `gen` (PCG64) is advanced accordingly."""
        st = pcg_state(gen)
        self._check(self.lib.ivhd_init_positions(self.h, st.ctypes.data_as(c_u64p), float(low), float(high)))
        pcg_store(gen, st)

    def set_connections(self, slot, edges, is_random, targets=None, scale=None):
        e = i32(edges).reshape(-1, 2)
        r = np.ascontiguousarray(is_random, dtype=np.uint8)
        t = None if targets is None else f64(targets)
        s = None if scale is None else f64(scale)
        self._check(self.lib.ivhd_set_connections(
            self.h, int(slot), ptr(e, ctypes.c_int32), ptr(r, ctypes.c_uint8),
            ptr(t, ctypes.c_double), ptr(s, ctypes.c_double), int(e.shape[0])))

    # ---------------------------------------------------------------- state
    def set_positions(self, y):
        y = f64(y)
        if y.shape != (self.m, self.dim):
            raise InvalidArgumentError(f"positions must be ({self.m}, {self.dim})")
        self._check(self.lib.ivhd_set_positions(self.h, y.ctypes.data_as(c_f64p)))

    def positions(self, out=None):
        out = np.empty((self.m, self.dim)) if out is None else out
        assert out.shape == (self.m, self.dim) and out.dtype == np.float64 and out.flags.c_contiguous
        self._check(self.lib.ivhd_get_positions(self.h, out.ctypes.data_as(c_f64p)))
        return out

    def deltas(self, out=None):
        out = np.empty((self.m, self.dim)) if out is None else out
        assert out.shape == (self.m, self.dim) and out.dtype == np.float64 and out.flags.c_contiguous
        self._check(self.lib.ivhd_get_deltas(self.h, out.ctypes.data_as(c_f64p)))
        return out

    def set_optimizer(self, params):
        self._check(self.lib.ivhd_set_optimizer(self.h, ctypes.byref(params)))

    def set_step_size(self, value):
        self._check(self.lib.ivhd_set_step_size(self.h, float(value)))

    def step_size(self):
        v = ctypes.c_double()
        self._check(self.lib.ivhd_get_step_size(self.h, ctypes.byref(v)))
        return v.value

    # ---------------------------------------------------------------- loops
    # Resolves the directions of degenerate random pairs when the device
    # pauses (degenerate.py): callable(slot, rows, entries) -> (rows,
    # entries, vecs) drawn from the run's generator; set by run_embedding's
    # session, which owns the connection lists and the generator.
    degenerate_resolver = None

    def _resolve(self, slot):
        n = ctypes.c_int64()
        self._check(self.lib.ivhd_degenerate_pending(self.h, 0, ctypes.byref(n), None, None))
        rows = np.empty(n.value, dtype=np.int32)
        ent = np.empty(n.value, dtype=np.int32)
        self._check(self.lib.ivhd_degenerate_pending(self.h, n.value, ctypes.byref(n),
                                                     rows.ctypes.data_as(c_i32p), ent.ctypes.data_as(c_i32p)))
        if self.degenerate_resolver is None:
            from .errors import DeviceError

            raise DeviceError("random pairs at zero distance need directions from the run's generator "
                              "(forces.py:167-174): use run_embedding / compute_forces, or set "
                              "DeviceEmbedding.degenerate_resolver")
        t_rows, t_ent, t_vec = self.degenerate_resolver(slot, rows, ent)
        t_rows, t_ent, t_vec = i32(t_rows), i32(t_ent), f64(t_vec)
        self._check(self.lib.ivhd_set_degenerate(self.h, len(t_rows), t_rows.ctypes.data_as(c_i32p),
                                                 t_ent.ctypes.data_as(c_i32p), t_vec.ctypes.data_as(c_f64p)))

    def run(self, slot, norm, c, n_iter):
        """Run n_iter iterations; returns (stress[], step[], done, diverged).
        An iteration that meets degenerate random pairs pauses on the device;
        the directions are drawn on the host and the iteration re-runs."""
        n_iter = int(n_iter)
        parts_s, parts_b, total = [], [], 0
        while True:
            left = n_iter - total
            stress = np.empty(max(left, 1))
            step = np.empty(max(left, 1))
            done = ctypes.c_int64(0)
            code = self.lib.ivhd_run(self.h, int(slot), _lib.NORM[norm], float(c), left,
                                     stress.ctypes.data_as(c_f64p), step.ctypes.data_as(c_f64p),
                                     ctypes.byref(done))
            d = done.value
            if code == _lib.PAUSED_DEGENERATE:
                parts_s.append(stress[:d])
                parts_b.append(step[:d])
                total += d
                self._resolve(slot)
                continue
            if code == _lib.ERR_DIVERGED:
                parts_s.append(stress[: d + 1])
                parts_b.append(step[: d + 1])
                return np.concatenate(parts_s), np.concatenate(parts_b), total + d, True
            self._check(code)
            parts_s.append(stress[:d])
            parts_b.append(step[:d])
            return np.concatenate(parts_s), np.concatenate(parts_b), total + d, False

    def compute_forces(self, slot, norm, c, y):
        y = f64(y)
        f = np.empty((self.m, self.dim))
        e = ctypes.c_double()
        for _ in range(2):
            code = self.lib.ivhd_compute_forces(self.h, int(slot), _lib.NORM[norm], float(c),
                                                y.ctypes.data_as(c_f64p), f.ctypes.data_as(c_f64p),
                                                ctypes.byref(e))
            if code != _lib.PAUSED_DEGENERATE:
                break
            self._resolve(slot)  # directions drawn on the host, then evaluate again
        self._check(code)
        return f, e.value

    def stress(self, slot, norm, c, y):
        y = f64(y)
        e = ctypes.c_double()
        self._check(self.lib.ivhd_stress(self.h, int(slot), _lib.NORM[norm], float(c),
                                         y.ctypes.data_as(c_f64p), ctypes.byref(e)))
        return e.value

    def synchronize(self):
        self._check(self.lib.ivhd_synchronize(self.h))

    def snapshot(self):
        self._check(self.lib.ivhd_snapshot(self.h))

    def restore(self):
        self._check(self.lib.ivhd_restore(self.h))

    # -------------------------------------------------------------- sharding
    def tiles(self):
        tv, nt = ctypes.c_int64(), ctypes.c_int64()
        self._check(self.lib.ivhd_tile_vertices(self.h, ctypes.byref(tv), ctypes.byref(nt)))
        return tv.value, nt.value

    def shard_set_range(self, v_begin, v_end):
        self._check(self.lib.ivhd_shard_set_range(self.h, int(v_begin), int(v_end)))

    def shard_buffers(self):
        y0, y1, p = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        fpv, cur = ctypes.c_int64(), ctypes.c_int()
        self._check(self.lib.ivhd_shard_buffers(self.h, ctypes.byref(y0), ctypes.byref(y1),
                                                ctypes.byref(fpv), ctypes.byref(p),
                                                ctypes.byref(cur)))
        return {"ybuf": (y0.value, y1.value), "floats_per_vertex": fpv.value,
                "partials": p.value, "cur": cur.value}

    def step_local(self, slot, norm, c):
        self._check(self.lib.ivhd_step_local(self.h, int(slot), _lib.NORM[norm], float(c)))

    def step_finalize(self):
        e, s, com = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        code = self.lib.ivhd_step_finalize(self.h, ctypes.byref(e), ctypes.byref(s),
                                           ctypes.byref(com))
        if code == _lib.ERR_DIVERGED:
            return e.value, s.value, bool(com.value), True
        self._check(code)
        return e.value, s.value, bool(com.value), False

    # fused peer exchange (include/ivhd_b200.h, ivhd_peer_*)
    def peer_export(self, world, rank):
        """Move the exchanged buffers to IPC-able memory; returns this rank's
        handle bytes (to be all-gathered in rank order)."""
        h = np.zeros(_lib.PEER_HANDLE_BYTES, dtype=np.uint8)
        self._check(self.lib.ivhd_peer_export(self.h, int(world), int(rank), h.ctypes.data_as(c_u8p)))
        return h.tobytes()

    def peer_import(self, handles):
        """handles: the ranks' peer_export bytes, in rank order."""
        buf = np.frombuffer(b"".join(handles), dtype=np.uint8).copy()
        self._check(self.lib.ivhd_peer_import(self.h, buf.ctypes.data_as(c_u8p)))

    def peer_import_local(self, devs):
        """In-process peers: the DeviceEmbedding of every rank, in rank order."""
        arr = (ctypes.c_void_p * len(devs))(*[d.h.value for d in devs])
        self._check(self.lib.ivhd_peer_import_local(self.h, arr))

    def peer_pull(self, barrier=True):
        """Complete the local replica with every peer's own range (ivhd_run
        does this at the end of each segment)."""
        self._check(self.lib.ivhd_peer_pull(self.h, int(bool(barrier))))

    def peer_halo(self):
        """(records, bytes) this rank stores into peers per iteration."""
        n, b = ctypes.c_int64(), ctypes.c_int64()
        self._check(self.lib.ivhd_peer_halo(self.h, ctypes.byref(n), ctypes.byref(b)))
        return n.value, b.value

    def gather_floor(self, slot=0, reps=10):
        """Device time (us) of one gather-only pass over the slot's connections:
        the column ids streamed and every neighbour position gathered, nothing
        else (ivhd_gather_floor) — the memory-system floor of one iteration."""
        us = ctypes.c_double()
        self._check(self.lib.ivhd_gather_floor(self.h, int(slot), int(reps), ctypes.byref(us)))
        return us.value

    def peer_set_timeout(self, seconds):
        """Peer failure detection: wait at most `seconds` for the other ranks'
        arrival flags, then fail with IVHD_ERR_PEER (DeviceError, status 5) instead of hanging."""
        self._check(self.lib.ivhd_peer_set_timeout(self.h, float(seconds)))

    # asynchronous sharded loop (include/ivhd_b200.h, ivhd_shard_*)
    def shard_begin(self, slot, c, n_iter):
        """Returns (index of the buffer holding the current positions, graph
        epoch — changes whenever previously captured launches went stale)."""
        self._n_shard = int(n_iter)
        cur, ep = ctypes.c_int(), ctypes.c_int64()
        self._check(self.lib.ivhd_shard_begin(self.h, int(slot), float(c), int(n_iter), ctypes.byref(cur),
                                              ctypes.byref(ep)))
        return cur.value, ep.value

    def shard_step(self, slot, norm):
        """Queue the local update; returns the device pointer of the buffer
        to all-gather (no host synchronisation)."""
        ptr_ = ctypes.c_uint64()
        self._check(self.lib.ivhd_shard_step(self.h, int(slot), _lib.NORM[norm], ctypes.byref(ptr_)))
        return ptr_.value

    def shard_finalize(self):
        self._check(self.lib.ivhd_shard_finalize(self.h))

    def shard_end(self):
        n = max(self._n_shard, 1)
        stress, step = np.empty(n), np.empty(n)
        done = ctypes.c_int64(0)
        code = self.lib.ivhd_shard_end(self.h, stress.ctypes.data_as(c_f64p), step.ctypes.data_as(c_f64p),
                                       ctypes.byref(done))
        if code == _lib.ERR_DIVERGED:
            d = done.value
            return stress[: d + 1], step[: d + 1], d, True
        self._check(code)
        return stress[: done.value], step[: done.value], done.value, False


__all__ = ["DeviceEmbedding", "c_i64p", "c_u8p"]
