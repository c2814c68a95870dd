"""Directions for degenerate random pairs (reference forces.py:158-174).

A connection with a nonzero target whose endpoints sit at exactly the same
position has no direction; the reference gives every such connection a unit
vector drawn from the run's generator — `rng.standard_normal((k, dim))` over
the degenerate connections in connection order, normalised, times w * t —
and adds it to the source row and subtracts it from the destination row.

On the GPU the draw stays on the host, where the run's numpy Generator
lives: the kernel reports each degenerate entry it meets as (row, entry
index within the row of the symmetrised CSR) and pauses the iteration
(ivhd_run returns IVHD_PAUSED_DEGENERATE, nothing committed).  `table`
maps those entries back to connection ids, makes exactly the reference's
draw, and returns the per-row table (both rows of every connection, with
opposite signs) that ivhd_set_degenerate uploads before the iteration is
re-run.  Measure-zero after a random initial layout; the tests force it.
"""

import numpy as np


def connection_of(row, k, src, dst, outdeg):
    """Connection id of entry k of `row`: the row lists its out-halves in
    connection order, then its in-halves in connection order (the CSR build,
    csrc/ivhd_capi.cu build_csr)."""
    if k < outdeg[row]:
        return int(np.flatnonzero(src == row)[k])
    return int(np.flatnonzero(dst == row)[k - outdeg[row]])


def table(rows, entries, src, dst, wt, rng, dim):
    """-> (rows, entries, vecs (n, dim)) for ivhd_set_degenerate, drawing from
    `rng` exactly as forces.py:167-171 does.  src/dst/wt: the active
    connection set (wt = w * t per connection, w including the scale)."""
    src = np.asarray(src)
    dst = np.asarray(dst)
    m = int(max(src.max(initial=-1), dst.max(initial=-1))) + 1
    outdeg = np.bincount(src, minlength=m)
    bad = np.unique([connection_of(int(r), int(k), src, dst, outdeg) for r, k in zip(rows, entries)])
    dirs = rng.standard_normal((bad.size, dim))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    vecs = dirs * np.asarray(wt, dtype=np.float64)[bad][:, None]
    t_rows, t_ent, t_vec = [], [], []
    for j, e in enumerate(bad):
        s, d = int(src[e]), int(dst[e])
        t_rows += [s, d]
        t_ent += [int(np.searchsorted(np.flatnonzero(src == s), e)),
                  int(outdeg[d] + np.searchsorted(np.flatnonzero(dst == d), e))]
        t_vec += [vecs[j], -vecs[j]]
    return (np.asarray(t_rows, dtype=np.int32), np.asarray(t_ent, dtype=np.int32),
            np.asarray(t_vec, dtype=np.float64).reshape(-1, dim))
