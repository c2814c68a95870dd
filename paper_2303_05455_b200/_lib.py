"""ctypes binding of libivhd_b200.so (declared in include/ivhd_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, the first call raises DeviceError.
"""

import ctypes
import os
import threading
import weakref

import numpy as np

from .errors import DeviceError, IvhdError, InvalidArgumentError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IVHD_B200_LIB", os.path.join(HERE, "libivhd_b200.so"))

OK, ERR_INVALID_ARG, ERR_CUDA, ERR_DIVERGED, ERR_STATE, ERR_PEER, PAUSED_DEGENERATE = range(7)
PEER_HANDLE_BYTES = 256
NORM = {"l2": 0, "l1": 1}
OPT_KIND = {"force-directed": 0, "sgd": 1, "momentum": 2, "nesterov": 3, "adam": 4, "adadelta": 5}

ABI_VERSION = 3
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_f64p = ctypes.POINTER(ctypes.c_double)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_u8p = ctypes.POINTER(ctypes.c_uint8)


class OptimizerParams(ctypes.Structure):
    """ivhd_optimizer_params."""

    _fields_ = [
        ("kind", ctypes.c_int32), ("auto_adapt", ctypes.c_int32), ("step", ctypes.c_double),
        ("a", ctypes.c_double), ("tau", ctypes.c_double), ("gamma1", ctypes.c_double),
        ("gamma2", ctypes.c_double), ("beta", ctypes.c_double), ("gamma_v", ctypes.c_double),
        ("gamma_s", ctypes.c_double), ("rho", ctypes.c_double), ("eps", ctypes.c_double),
    ]


# name -> (restype, argtypes); exactly the symbols include/ivhd_b200.h declares
SIGNATURES = {
    "ivhd_abi_version": (ctypes.c_int, []),
    "ivhd_global_error": (ctypes.c_char_p, []),
    "ivhd_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int64,
                                   ctypes.c_int, ctypes.c_uint64]),
    "ivhd_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "ivhd_last_error": (ctypes.c_char_p, [ctypes.c_void_p]),
    "ivhd_set_graph": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_i32p, ctypes.c_int64,
                                      ctypes.c_int, c_i32p, ctypes.c_int]),
    "ivhd_init_positions": (ctypes.c_int, [ctypes.c_void_p, c_u64p, ctypes.c_double, ctypes.c_double]),
    "ivhd_set_graph_sampled": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_i32p, ctypes.c_int64,
                                              ctypes.c_int, ctypes.c_int, c_u64p, c_i32p]),
    "ivhd_shard_begin": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64,
                                        ctypes.POINTER(ctypes.c_int), c_i64p]),
    "ivhd_shard_step": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, c_u64p]),
    "ivhd_shard_finalize": (ctypes.c_int, [ctypes.c_void_p]),
    "ivhd_shard_end": (ctypes.c_int, [ctypes.c_void_p, c_f64p, c_f64p, c_i64p]),
    "ivhd_peer_export": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, c_u8p]),
    "ivhd_peer_import": (ctypes.c_int, [ctypes.c_void_p, c_u8p]),
    "ivhd_peer_import_local": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "ivhd_peer_pull": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "ivhd_degenerate_pending": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, c_i64p, c_i32p, c_i32p]),
    "ivhd_set_degenerate": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, c_i32p, c_i32p, c_f64p]),
    "ivhd_peer_halo": (ctypes.c_int, [ctypes.c_void_p, c_i64p, c_i64p]),
    "ivhd_peer_set_timeout": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double]),
    "ivhd_gather_floor": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, c_f64p]),
    "ivhd_set_connections": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_i32p, c_u8p, c_f64p,
                                            c_f64p, ctypes.c_int64]),
    "ivhd_set_positions": (ctypes.c_int, [ctypes.c_void_p, c_f64p]),
    "ivhd_get_positions": (ctypes.c_int, [ctypes.c_void_p, c_f64p]),
    "ivhd_get_deltas": (ctypes.c_int, [ctypes.c_void_p, c_f64p]),
    "ivhd_set_optimizer": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(OptimizerParams)]),
    "ivhd_set_step_size": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double]),
    "ivhd_get_step_size": (ctypes.c_int, [ctypes.c_void_p, c_f64p]),
    "ivhd_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                ctypes.c_int64, c_f64p, c_f64p, c_i64p]),
    "ivhd_compute_forces": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_double, c_f64p, c_f64p, c_f64p]),
    "ivhd_stress": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                   c_f64p, c_f64p]),
    "ivhd_synchronize": (ctypes.c_int, [ctypes.c_void_p]),
    "ivhd_snapshot": (ctypes.c_int, [ctypes.c_void_p]),
    "ivhd_restore": (ctypes.c_int, [ctypes.c_void_p]),
    "ivhd_tile_vertices": (ctypes.c_int, [ctypes.c_void_p, c_i64p, c_i64p]),
    "ivhd_shard_set_range": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64]),
    "ivhd_shard_buffers": (ctypes.c_int, [ctypes.c_void_p, c_u64p, c_u64p, c_i64p, c_u64p,
                                          ctypes.POINTER(ctypes.c_int)]),
    "ivhd_step_local": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_double]),
    "ivhd_step_finalize": (ctypes.c_int, [ctypes.c_void_p, c_f64p, c_f64p,
                                          ctypes.POINTER(ctypes.c_int)]),
    "ivhd_knn_last_error": (ctypes.c_char_p, []),
    "ivhd_metrics_last_error": (ctypes.c_char_p, []),
    "ivhd_neighbor_hit": (ctypes.c_int, [ctypes.c_int, c_f64p, ctypes.c_int64, ctypes.c_int32, c_i32p,
                                         ctypes.c_int32, c_f64p, c_i32p]),
    "ivhd_host_alloc": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]),
    "ivhd_host_free": (ctypes.c_int, [ctypes.c_void_p]),
    "ivhd_rank_matrix": (ctypes.c_int, [ctypes.c_int, c_f64p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                        c_i64p]),
    "ivhd_pair_ranks": (ctypes.c_int, [ctypes.c_int, c_f64p, ctypes.c_int64, ctypes.c_int32, c_i64p, c_i64p,
                                       ctypes.c_int64, c_i64p]),
    "ivhd_curve_pass": (ctypes.c_int, [ctypes.c_int, c_f64p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                       c_f64p, ctypes.c_int32, c_i32p, ctypes.c_int32, c_i32p, ctypes.c_int32,
                                       c_i64p, c_i64p, c_i64p, c_i64p, c_i64p]),
    "ivhd_knn_build": (ctypes.c_int, [ctypes.c_int, c_f64p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_int32, c_i32p, c_f64p, c_f64p]),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the CDLL; raises DeviceError if it is absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"CUDA library not built: {LIB_PATH} is missing "
                    "(run `python -m paper_2303_05455_b200.build`)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.ivhd_abi_version() != ABI_VERSION:
                raise DeviceError("libivhd_b200.so ABI version mismatch")
            _lib = lib
        return _lib


def ptr(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype)) if a is not None else None


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class StatusError(IvhdError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def check(code, ctx_handle=None):
    """Map an ivhd_status to the reference's exception classes."""
    if code == OK:
        return
    lib = load()
    msg = (lib.ivhd_last_error(ctx_handle) if ctx_handle else lib.ivhd_global_error()) or b""
    msg = msg.decode(errors="replace")
    if code == ERR_INVALID_ARG:
        raise InvalidArgumentError(msg)
    if code == ERR_DIVERGED:
        raise StatusError(code, msg)
    raise DeviceError(f"ivhd status {code}: {msg}")


class PinnedPool:
    """Page-locked host buffers for result arrays (positions, deltas), recycled
    when the arrays that use them are garbage-collected.

    A run's device -> host copies land directly in them at full link rate, and
    a recycled buffer has no first-touch page faults (fresh 22 MB arrays cost
    ~5 ms each at C3).  Pinned bytes (handed out + pooled) stay below
    `cap_bytes` (default min(16 GiB, 1/8 of physical memory)); pooled buffers of
    other sizes are released to make room.  Arrays below 1 MiB, above
    `max_bytes`, or that do not fit the cap are plain numpy allocations.
    """

    def __init__(self, max_bytes=4 << 30, cap_bytes=None):
        if cap_bytes is None:
            try:
                phys = os.sysconf("SC_PHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
            except (ValueError, OSError, AttributeError):
                phys = 16 << 30
            cap_bytes = min(16 << 30, phys // 8)
        self.max_bytes = max_bytes
        self.cap_bytes = cap_bytes
        self._free = {}  # nbytes -> [address]
        self._outstanding = 0
        self._pooled = 0
        self._lock = threading.Lock()

    def empty(self, shape, device=0):
        n = int(np.prod(shape))
        nbytes = n * 8
        if nbytes < (1 << 20) or nbytes > self.max_bytes:
            return np.empty(shape)
        with self._lock:
            lst = self._free.get(nbytes)
            if lst:
                addr = lst.pop()
                self._pooled -= nbytes
            else:
                # make room by releasing pooled buffers of other sizes
                for size in sorted(self._free, reverse=True):
                    while self._free[size] and self._outstanding + self._pooled + nbytes > self.cap_bytes:
                        load().ivhd_host_free(ctypes.c_void_p(self._free[size].pop()))
                        self._pooled -= size
                if self._outstanding + self._pooled + nbytes > self.cap_bytes:
                    return np.empty(shape)
                out = ctypes.c_void_p()
                if load().ivhd_host_alloc(int(device), nbytes, ctypes.byref(out)) != OK or not out.value:
                    return np.empty(shape)
                addr = out.value
            self._outstanding += nbytes
        buf = (ctypes.c_char * nbytes).from_address(addr)
        weakref.finalize(buf, self._release, addr, nbytes)
        return np.frombuffer(buf, dtype=np.float64, count=n).reshape(shape)

    def _release(self, addr, nbytes):
        with self._lock:
            self._outstanding -= nbytes
            self._pooled += nbytes
            self._free.setdefault(nbytes, []).append(addr)


pinned = PinnedPool()
