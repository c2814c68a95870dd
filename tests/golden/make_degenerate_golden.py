"""Golden forces from the REFERENCE for random pairs at zero distance
(forces.py:158-174: a unit direction per degenerate connection from
rng.standard_normal((k, dim)) in connection order, magnitude w * t).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_degenerate_golden.py

Cases: binary 2-D with a seeded generator, the same with rng=None (the
reference then uses default_rng(0)), 3-D, and scaled weights with
euclidean-style targets; several coincident points, some pairs listed in
both directions and one duplicated connection.  Stored per case: positions,
connection arrays, c, the seed (-1 = None), the reference's forces and stress.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def case(rng, dim, m=40, n_rand=30, weighted=False):
    y = rng.uniform(-1, 1, (m, dim))
    y[5] = y[3]          # coincident points
    y[9] = y[3]
    y[17] = y[11]
    y[30] = y[22]
    nn = np.column_stack([np.arange(m), (np.arange(m) + 1) % m])
    rn = np.array([[3, 5], [9, 3], [5, 9], [11, 17], [17, 11], [22, 30], [22, 30], [0, 7]] +
                  [[int(a), int(b)] for a, b in rng.integers(0, m, size=(n_rand, 2)) if a != b])
    edges = np.vstack([nn, rn]).astype(np.int32)
    is_random = np.r_[np.zeros(len(nn), bool), np.ones(len(rn), bool)]
    if weighted:
        targets = np.where(is_random, rng.uniform(0.2, 1.0, len(edges)), rng.uniform(0.0, 0.3, len(edges)))
        targets[len(nn)] = 0.7
        scale = rng.uniform(0.5, 2.0, len(edges))
    else:
        targets = is_random.astype(np.float64)
        scale = None
    return y, edges, targets, is_random, scale


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    from ivhd import forces as F

    rng = np.random.default_rng(11)
    out = {}
    specs = [("bin2_seed", 2, False, 7), ("bin2_none", 2, False, -1), ("bin3_seed", 3, False, 3),
             ("w2_seed", 2, True, 5)]
    for k, (name, dim, weighted, seed) in enumerate(specs):
        y, edges, targets, is_random, scale = case(rng, dim, weighted=weighted)
        conn = F.ConnectionSet(edges, targets, is_random, scale)
        c = 0.1
        gen = None if seed < 0 else np.random.default_rng(seed)
        f, e = F.compute_forces(y, conn, c, F.NORM_L2, rng=gen, with_stress=True)
        p = f"d{k}_"
        out.update({p + "name": np.array(name), p + "Y": y, p + "edges": edges, p + "targets": targets,
                    p + "is_random": is_random, p + "scale": np.zeros(0) if scale is None else scale,
                    p + "c": np.float64(c), p + "seed": np.int64(seed), p + "force": f,
                    p + "stress": np.float64(e)})
    out["n_cases"] = np.int64(len(specs))
    np.savez_compressed(os.path.join(HERE, "degenerate_cases.npz"), **out)
    print("wrote", len(specs), "cases")


if __name__ == "__main__":
    main()
