import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_2303_05455_b200 as P
from paper_2303_05455_b200.device import DeviceEmbedding

rng = np.random.default_rng(0)
for m, deg in ((30, 3), (30, 5), (100, 3), (300, 4)):
    src = np.repeat(np.arange(m), deg)
    dst = (src + rng.integers(1, m, src.size)) % m
    conn = O.Connections(src, dst, np.zeros(src.size), np.zeros(src.size, bool))
    Y = rng.uniform(-1, 1, (m, 2))
    fr, er = O.forces(Y, conn, 0.1, with_stress=True)
    with DeviceEmbedding(m, 2) as dev:
        dev.set_connections(0, np.column_stack([src, dst]), np.zeros(src.size, np.uint8))
        f, e = dev.compute_forces(0, "l2", 0.1, Y)
    row_ptr, other, cidx = O.symmetrise(conn, m)
    d = np.abs(f - fr).max(axis=1)
    bad = np.flatnonzero(d > 1e-4)
    print(f"m={m} deg={deg} entries={row_ptr[-1]} stress {e:.6f} vs {er:.6f}; bad rows {bad.size}")
    P_ = 12
    for r in bad[:12]:
        rs, re = row_ptr[r], row_ptr[r + 1]
        print(f"  row {r} entries [{rs},{re}) diag [{rs + r},{re - 1 + r}] threads {(rs + r)//P_}..{(re - 1 + r)//P_}  got {f[r]} want {fr[r]}")
