"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference IVHD loop.

Not part of the product: imported only by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline leg (see oracle/__init__.py).

Every function cites the reference lines it restates (paths relative to
/root/reference/pkg/src/ivhd/).  Arithmetic is float64 throughout, like the
reference.  Two force formulations are provided:

* `forces()`      — the reference's two-phase edge-list evaluation
                    (per-connection component, then a fixed-order bincount);
* `csr_forces()`  — the vertex-centric symmetrised-CSR formulation the CUDA
                    kernel implements (each connection listed in the rows of
                    both endpoints).  It agrees with `forces()` to ~1e-16 in
                    float64, which is the math contract of the kernel.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

L1 = "l1"
L2 = "l2"

OPTIMIZERS = ("force-directed", "sgd", "momentum", "nesterov", "adam", "adadelta")
ALPHA_DEFAULT = {"sgd": 0.1, "momentum": 0.02, "nesterov": 0.02, "adam": 0.05, "adadelta": 1.0}


class OracleDiverged(Exception):
    """Raised like NumericalDivergenceError (engine.py:373-377)."""

    def __init__(self, iteration, positions, stress):
        super().__init__(f"diverged at iteration {iteration}")
        self.iteration = iteration
        self.positions = positions
        self.stress = stress


# --------------------------------------------------------------- connections


@dataclass
class Connections:
    """Directed connection list; mirrors ConnectionSet (forces.py:20-67)."""

    src: np.ndarray
    dst: np.ndarray
    target: np.ndarray
    rand: np.ndarray
    scale: np.ndarray | None = None

    def __len__(self):
        return int(self.src.shape[0])

    def weights(self, c):
        # forces.py:55-59 — c on random pairs, 1 on nn pairs, times scale
        w = np.where(self.rand, float(c), 1.0)
        return w if self.scale is None else w * self.scale

    @classmethod
    def from_reference(cls, conn):
        e = np.asarray(conn.edges)
        sc = None if conn.scale is None else np.asarray(conn.scale, dtype=np.float64)
        return cls(e[:, 0].astype(np.int64), e[:, 1].astype(np.int64),
                   np.asarray(conn.targets, dtype=np.float64),
                   np.asarray(conn.is_random, dtype=bool), sc)


def init_layout(m, dim, rng):
    """engine.py:124-129: U[-1,1]^(m,dim) from the run generator."""
    return rng.uniform(-1.0, 1.0, size=(m, dim))


def sample_rn(m, nn_sets, rn, rng):
    """engine.py:132-146: uniform over non-self, non-nn ids, by rejection.

    The draw order (one block of m*rn integers, then re-draws of the rejected
    slots in row-major order) is what keeps the PCG64 stream identical.
    """
    nn_sets = np.asarray(nn_sets)
    if m <= nn_sets.shape[1] + rn:
        raise ValueError("graph too small for nn + rn")
    draw = rng.integers(0, m, size=(m, rn))
    me = np.arange(m)[:, None]
    while True:
        clash = draw == me
        for col in range(nn_sets.shape[1]):
            clash |= draw == nn_sets[:, col][:, None]
        n_bad = int(clash.sum())
        if n_bad == 0:
            return draw.astype(np.int32)
        draw[clash] = rng.integers(0, m, size=n_bad)


def build_connections(nn_sets, rn_assign, nn_targets=None, rn_targets=None):
    """engine.py:225-262: nn block (i, nn_sets[i,c]) i-major, then rn block."""
    m, ncols = nn_sets.shape
    rn = rn_assign.shape[1]
    src = np.concatenate([np.repeat(np.arange(m), ncols), np.repeat(np.arange(m), rn)])
    dst = np.concatenate([nn_sets.reshape(-1), rn_assign.reshape(-1)]).astype(np.int64)
    if nn_targets is None:
        nn_targets = np.zeros(m * ncols)
    if rn_targets is None:
        rn_targets = np.ones(m * rn)
    target = np.concatenate([nn_targets, rn_targets]).astype(np.float64)
    rand = np.zeros(src.shape[0], dtype=bool)
    rand[m * ncols:] = True
    return Connections(src.astype(np.int64), dst, target, rand)


def rnn_keep_mask(nn_src, nn_dst, nn_sets, helper_neighbors):
    """engine.py:289-309: keep (i,j) iff i in helper-kNN(j); orphans keep col 0."""
    hits = (helper_neighbors[nn_dst] == nn_src[:, None]).any(axis=1)
    m, ncols = nn_sets.shape
    per_row = hits.reshape(m, ncols).copy()
    lonely = ~per_row.any(axis=1)
    per_row[lonely, 0] = True
    return per_row.reshape(-1)


def filtered_connections(full, nn_sets, helper_neighbors):
    """engine.py:270-286: RNN-filtered nn part with per-edge budget scale."""
    m, ncols = nn_sets.shape
    n_nn = m * ncols
    keep = rnn_keep_mask(full.src[:n_nn], full.dst[:n_nn], nn_sets, helper_neighbors)
    kept_per = keep.reshape(m, ncols).sum(axis=1)
    nn_scale = (ncols / kept_per)[full.src[:n_nn][keep]]
    rn_sl = slice(n_nn, len(full))
    return Connections(
        np.concatenate([full.src[:n_nn][keep], full.src[rn_sl]]),
        np.concatenate([full.dst[:n_nn][keep], full.dst[rn_sl]]),
        np.concatenate([full.target[:n_nn][keep], full.target[rn_sl]]),
        np.concatenate([np.zeros(int(keep.sum()), bool), np.ones(len(full) - n_nn, bool)]),
        np.concatenate([nn_scale, np.ones(len(full) - n_nn)]),
    )


# -------------------------------------------------------------------- forces


def _dist(diff, norm):
    if norm == L2:
        return np.sqrt((diff * diff).sum(axis=1))
    if norm == L1:
        return np.abs(diff).sum(axis=1)
    raise ValueError(f"unknown norm {norm!r}")


def stress(Y, conn, c, norm=L2):
    """forces.py:78-83: E = sum_conn w (t - d)^2."""
    d = _dist(Y[conn.src] - Y[conn.dst], norm)
    r = conn.target - d
    return float(np.sum(conn.weights(c) * r * r))


def components(Y, conn, c, norm, lo=0, hi=None):
    """forces.py:86-125 (phase 1) over connections [lo, hi).

    Returns (comp (n,dim), energy (n,), degenerate mask (n,)).
    """
    hi = len(conn) if hi is None else hi
    sl = slice(lo, hi)
    w = conn.weights(c)[sl]
    t = conn.target[sl]
    diff = Y[conn.src[sl]] - Y[conn.dst[sl]]
    if norm == L1:
        d = np.abs(diff).sum(axis=1)
        r = t - d
        comp = np.sign(diff) * (w * r)[:, None]
        degen = np.zeros(hi - lo, dtype=bool)
    elif norm == L2:
        d = np.sqrt((diff * diff).sum(axis=1))
        r = t - d
        at_zero = d == 0.0
        with np.errstate(invalid="ignore", divide="ignore"):
            phi = np.where(t == 0.0, -w, w * r / np.where(at_zero, 1.0, d))
        degen = at_zero & (t != 0.0)
        phi[degen] = 0.0
        comp = diff * phi[:, None]
    else:
        raise ValueError(f"unknown norm {norm!r}")
    return comp, w * r * r, degen


def accumulate(comp, conn, m):
    """forces.py:128-136 (phase 2): fixed-order bincount per axis."""
    out = np.empty((m, comp.shape[1]))
    for a in range(comp.shape[1]):
        out[:, a] = (np.bincount(conn.src, weights=comp[:, a], minlength=m)
                     - np.bincount(conn.dst, weights=comp[:, a], minlength=m))
    return out


def forces(Y, conn, c, norm=L2, rng=None, threads=1, with_stress=False):
    """forces.py:139-181: force = -1/2 grad E, degenerate rn pairs get a
    seeded random unit direction of magnitude w*t drawn in connection order.
    `threads` splits phase 1 into slabs like forces.py:151-163."""
    m, dim = Y.shape
    n = len(conn)
    if threads > 1 and n >= 4 * threads:
        cuts = np.linspace(0, n, threads + 1, dtype=int)
        with ThreadPoolExecutor(max_workers=threads) as pool:
            parts = list(pool.map(lambda k: components(Y, conn, c, norm, cuts[k], cuts[k + 1]),
                                  range(threads)))
        comp = np.concatenate([p[0] for p in parts]) if parts else np.empty((0, dim))
        energy = np.concatenate([p[1] for p in parts])
        degen = np.concatenate([p[2] for p in parts])
    else:
        comp, energy, degen = components(Y, conn, c, norm)
    bad = np.flatnonzero(degen)
    if bad.size:
        rng = np.random.default_rng(0) if rng is None else rng
        u = rng.standard_normal((bad.size, dim))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        comp[bad] = u * (conn.weights(c)[bad] * conn.target[bad])[:, None]
    f = accumulate(comp, conn, m)
    if with_stress:
        return f, float(np.sum(energy))
    return f


# ------------------------------------------------- vertex-centric formulation


def symmetrise(conn, m):
    """The kernel's symmetrised CSR: row i lists every connection incident to
    i — first the connections where i is the source (in connection order),
    then those where i is the destination (in connection order).  Returns
    (row_ptr (m+1,), other (2L,), conn_index (2L,))."""
    n = len(conn)
    rows = np.concatenate([conn.src, conn.dst])
    other = np.concatenate([conn.dst, conn.src])
    cidx = np.concatenate([np.arange(n), np.arange(n)])
    order = np.argsort(rows, kind="stable")
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=m), out=row_ptr[1:])
    return row_ptr, other[order], cidx[order]


def csr_forces(Y, csr, conn, c, norm=L2):
    """f_i = sum_{e in row i} phi_e (y_i - y_o(e)); E = 1/2 sum_i sum_e w(t-d)^2.

    Degenerate (d == 0, t != 0) L2 rows contribute zero force here (the
    reference draws a random direction for them; measure-zero)."""
    row_ptr, other, cidx = csr
    m = Y.shape[0]
    rows = np.repeat(np.arange(m), np.diff(row_ptr))
    diff = Y[rows] - Y[other]
    w = conn.weights(c)[cidx]
    t = conn.target[cidx]
    if norm == L2:
        d = np.sqrt((diff * diff).sum(axis=1))
        with np.errstate(invalid="ignore", divide="ignore"):
            phi = np.where(t == 0.0, -w, np.where(d == 0.0, 0.0, w * (t - d) / np.where(d == 0.0, 1.0, d)))
        contrib = diff * phi[:, None]
    else:
        d = np.abs(diff).sum(axis=1)
        contrib = np.sign(diff) * (w * (t - d))[:, None]
    f = np.zeros_like(Y)
    for a in range(Y.shape[1]):
        f[:, a] = np.bincount(rows, weights=contrib[:, a], minlength=m)
    return f, 0.5 * float(np.sum(w * (t - d) ** 2))


# ---------------------------------------------------------------- optimizers


def make_state(kind, m, dim, a=0.99, b=0.002, tau=None, gamma1=1.1, gamma2=0.9,
               auto_adapt=True, alpha=None, beta=0.9, gamma_v=0.9, gamma_s=0.999,
               rho=0.95, eps=1e-8):
    """optim.py:95-256: per-kind state dict (zeros) plus hyper-parameters."""
    if kind not in OPTIMIZERS:
        raise ValueError(f"unknown optimizer {kind!r}")
    st = {"kind": kind}
    zeros = lambda: np.zeros((m, dim))  # noqa: E731
    if kind == "force-directed":
        st.update(a=a, b=b, tau=1e-3 * m if tau is None else tau, g1=gamma1, g2=gamma2,
                  adapt=auto_adapt, delta=zeros(), rolled_back=False)
    else:
        st["alpha"] = ALPHA_DEFAULT[kind] if alpha is None else alpha
        if kind in ("momentum", "nesterov"):
            st.update(beta=beta, vel=zeros())
        elif kind == "adam":
            st.update(gv=gamma_v, gs=gamma_s, eps=eps, v=zeros(), s=zeros(), t=0)
        elif kind == "adadelta":
            st.update(rho=rho, eps=eps, sg=zeros(), sd=zeros())
    return st


def step_size(st):
    """optim.py:106-108 / 133-135 …: b for FD, alpha (or scale) otherwise."""
    return st["b"] if st["kind"] == "force-directed" else st["alpha"]


def lookahead(st, Y):
    """optim.py:110, 174-175: Nesterov evaluates forces at y + beta v."""
    if st["kind"] == "nesterov":
        return Y + st["beta"] * st["vel"]
    return Y


def optimizer_step(st, Y, force):
    """optim.py:80-263 incl. step_optimizer: grad = -2 force for the gradient
    kinds; force-directed consumes the force and may roll back."""
    kind = st["kind"]
    if kind == "force-directed":
        old = st["delta"]
        new = st["a"] * old + st["b"] * force
        st["delta"] = new
        st["rolled_back"] = False
        if st["adapt"]:
            # optim.py:80-92
            d_t = float(np.sum(new * new) - np.sum(old * old))
            if d_t > st["tau"]:
                st["b"] *= st["g2"]
                st["rolled_back"] = True
            elif d_t < -st["tau"]:
                st["b"] *= st["g1"]
                st["rolled_back"] = True
            if st["rolled_back"]:
                return Y
        return Y + new
    g = -2.0 * force
    if kind == "sgd":
        return Y - st["alpha"] * g
    if kind in ("momentum", "nesterov"):
        st["vel"] = st["beta"] * st["vel"] - st["alpha"] * g
        return Y + st["vel"]
    if kind == "adam":
        st["t"] += 1
        st["v"] = st["gv"] * st["v"] + (1.0 - st["gv"]) * g
        st["s"] = st["gs"] * st["s"] + (1.0 - st["gs"]) * g * g
        vh = st["v"] / (1.0 - st["gv"] ** st["t"])
        sh = st["s"] / (1.0 - st["gs"] ** st["t"])
        return Y - st["alpha"] * vh / (st["eps"] + np.sqrt(sh))
    # adadelta
    st["sg"] = st["rho"] * st["sg"] + (1.0 - st["rho"]) * g * g
    step = -st["alpha"] * np.sqrt(st["sd"] + st["eps"]) / np.sqrt(st["sg"] + st["eps"]) * g
    st["sd"] = st["rho"] * st["sd"] + (1.0 - st["rho"]) * step * step
    return Y + step


# ------------------------------------------------------------------ the loop


class OracleRun:
    """Replay of engine.run_embedding (engine.py:312-414) without observers.

    Consumes one PCG64 stream in the reference order (engine.py:165, 214-215,
    264-268, forces.py:167-171) so Y0 and the rn sample are bit-identical to
    the reference's.  `step()` performs one loop iteration and returns a
    record dict {iteration, force, positions, stress, b}.
    """

    def __init__(self, neighbors, nn=3, rn=1, c=0.1, iterations=2500, seed=0,
                 optimizer="force-directed", target_dim=2, l1_final_steps=0,
                 rnn_final_steps=0, rn_resample_period=0, helper_neighbors=None,
                 integrator=None, opt=None, threads=1, distance_mode="binary",
                 distances=None, data=None, normalize_targets=True):
        neighbors = np.asarray(neighbors)
        self.m = neighbors.shape[0]
        self.c = c
        self.rn = rn
        self.total = iterations
        self.threads = threads
        self.rng = np.random.default_rng(seed)
        self.nn_sets = neighbors[:, :min(nn, neighbors.shape[1])]
        self.helper = helper_neighbors
        self.euclid = distance_mode == "euclidean"
        self.distances = distances
        self.data = None if data is None else np.asarray(data, dtype=np.float64)
        self.normalize = normalize_targets
        self.tscale = None
        self.Y = init_layout(self.m, target_dim, self.rng)
        self.rn_assign = sample_rn(self.m, self.nn_sets, rn, self.rng)
        self._rebuild()
        kw = dict(integrator or {})
        kw.update(opt or {})
        self.opt = make_state(optimizer, self.m, target_dim, **kw)
        self.l1_from = iterations - l1_final_steps if l1_final_steps > 0 else None
        self.rnn_from = iterations - rnn_final_steps if rnn_final_steps > 0 else None
        self.period = rn_resample_period
        self.it = 0
        self.trace_stress = []
        self.trace_b = []

    def _rebuild(self):
        if not self.euclid:
            self.full = build_connections(self.nn_sets, self.rn_assign)
        else:
            # engine.py:229-253: stored kNN distances for nn pairs, feature-space
            # distances for rn pairs, both scaled once by 1/max
            ncols = self.nn_sets.shape[1]
            nn_t = np.asarray(self.distances)[:, :ncols].reshape(-1).astype(np.float64)
            src = np.repeat(np.arange(self.m), self.rn_assign.shape[1])
            diff = self.data[src] - self.data[self.rn_assign.reshape(-1)]
            rn_t = np.sqrt((diff * diff).sum(axis=1))
            if self.normalize:
                if self.tscale is None:
                    peak = max(float(nn_t.max(initial=0.0)), float(rn_t.max(initial=0.0)))
                    self.tscale = 1.0 / peak if peak > 0 else 1.0
                nn_t = nn_t * self.tscale
                rn_t = rn_t * self.tscale
            self.full = build_connections(self.nn_sets, self.rn_assign, nn_t, rn_t)
        self._filtered = None

    def filtered(self):
        if self._filtered is None:
            self._filtered = filtered_connections(self.full, self.nn_sets, self.helper)
        return self._filtered

    def step(self):
        it = self.it
        if self.period > 0 and it > 0 and it % self.period == 0:
            # engine.py:347-349
            self.rn_assign = sample_rn(self.m, self.nn_sets, self.rn, self.rng)
            self._rebuild()
        rnn_on = self.rnn_from is not None and it >= self.rnn_from
        l1_on = self.l1_from is not None and it >= self.l1_from
        conn = self.filtered() if rnn_on else self.full
        norm = L1 if l1_on else L2
        ev = lookahead(self.opt, self.Y)
        if ev is self.Y:
            f, e = forces(ev, conn, self.c, norm, rng=self.rng, threads=self.threads,
                          with_stress=True)
        else:
            f = forces(ev, conn, self.c, norm, rng=self.rng, threads=self.threads)
            e = stress(self.Y, conn, self.c, norm)
        new = optimizer_step(self.opt, self.Y, f)
        if not np.isfinite(new).all():
            raise OracleDiverged(it, self.Y, e)
        self.Y = new
        self.it += 1
        self.trace_stress.append(e)
        self.trace_b.append(step_size(self.opt))
        return {"iteration": it, "force": f, "positions": new, "stress": e,
                "b": step_size(self.opt)}

    def run(self, n=None):
        n = self.total - self.it if n is None else n
        for _ in range(n):
            self.step()
        return self.Y


# ------------------------------------------------------------- rank curves
# Restatement of metrics.py:57-110 (distance blocks, rank rule) and
# metrics.py:149-182 (`_curve_pass`), for small M (the full M x M rank
# matrices are materialised).  Checker for ivhd_curve_pass.


def _sq_dist_matrix(Z):
    """metrics.py:76-84: max((|a|^2 + |b|^2) - 2 a.b, 0)."""
    sq = np.einsum("ij,ij->i", Z, Z)
    D = sq[:, None] + sq[None, :] - 2.0 * (Z @ Z.T)
    np.maximum(D, 0.0, out=D)
    return D


def _ranks(D):
    """metrics.py:103-113: rank 1..M-1 by (distance, index), self = 0."""
    m = D.shape[0]
    D = np.array(D, dtype=np.float64)
    D[np.arange(m), np.arange(m)] = np.inf
    idx = np.broadcast_to(np.arange(m), (m, m))
    order = np.lexsort((idx, D), axis=1)
    ranks = np.empty((m, m), dtype=np.int64)
    np.put_along_axis(ranks, order, np.broadcast_to(np.arange(1, m + 1), (m, m)), axis=1)
    ranks[np.arange(m), np.arange(m)] = 0
    return ranks, order


def curve_pass(X, Y, labels, k_max, report_ks, x_precomputed=False):
    """metrics.py:149-182 -> (agree[0..k_max], same_ld, same_hd, trust_pen, cont_pen)."""
    m = X.shape[0]
    hd, hd_order = _ranks(X if x_precomputed else _sq_dist_matrix(X))
    ld, ld_order = _ranks(_sq_dist_matrix(Y))
    peak = np.maximum(hd, ld)
    peak[np.arange(m), np.arange(m)] = m
    agree = np.bincount(peak.ravel(), minlength=m + 1)[: k_max + 1].astype(np.int64)
    same_ld = same_hd = None
    if labels is not None:
        own = labels[:, None]
        same_ld = (labels[ld_order[:, :k_max]] == own).sum(axis=0)
        same_hd = (labels[hd_order[:, :k_max]] == own).sum(axis=0)
    trust, cont = {}, {}
    for k in report_ks:
        trust[k] = int((hd[(ld <= k) & (hd > k)] - k).sum())
        cont[k] = int((ld[(hd <= k) & (hd > 0) & (ld > k)] - k).sum())
    return agree, same_ld, same_hd, trust, cont
