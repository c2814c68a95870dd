"""Golden rank-curve values from the REFERENCE `ivhd.metrics` (rnx_curve,
gnn_curve, trust_continuity, evaluate_embedding; metrics.py:149-251, 351-380)
for tests/test_gpu_metrics.py and tests/test_oracle_golden.py.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_curves_golden.py

Inputs are regenerated from seeds by `curve_inputs()`; only the reference's
outputs (integer-derived curves, AUCs and trust/continuity values) are stored.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "curves.npz")


def curve_inputs():
    """name -> (X, Y, labels, k_max, report_ks, x_precomputed)."""
    out = {}
    # 10-cluster mixture in 20-D, Y = noisy 2-D projection (imperfect embedding)
    rng = np.random.default_rng(31)
    c = rng.standard_normal((10, 20)) * 2.0
    lab = rng.integers(0, 10, 600)
    X = c[lab] + rng.standard_normal((600, 20))
    Y = X[:, :2] + 0.7 * rng.standard_normal((600, 2))
    out["mix20_600"] = (X, Y, lab, None, (5, 15, 50, 100), False)
    # 50-D, 3-D embedding, default k_max clipped at 1000
    rng = np.random.default_rng(32)
    c = rng.standard_normal((6, 50)) * 1.5
    lab = rng.integers(0, 6, 1500)
    X = c[lab] + rng.standard_normal((1500, 50))
    Y = X[:, :3] + 0.3 * rng.standard_normal((1500, 3))
    out["mix50_1500_d3"] = (X, Y, lab, None, (15, 50, 100), False)
    # precomputed source distances (evaluate_embedding x_precomputed)
    rng = np.random.default_rng(33)
    X = rng.standard_normal((300, 8))
    D = np.sqrt(((X[:, None, :] - X[None, :, :]) ** 2).sum(-1))
    Y = X[:, :2] + 0.5 * rng.standard_normal((300, 2))
    lab = (X[:, 0] > 0).astype(np.int64) + 2 * (X[:, 1] > 0)
    out["precomp_300"] = (D, Y, lab, 120, (10, 40), True)
    # integer lattices: exact distance ties in both spaces (index tie rule)
    g = np.arange(20, dtype=np.float64)
    Y = np.stack(np.meshgrid(g, g, indexing="ij"), -1).reshape(-1, 2)
    X = np.concatenate([Y, (Y[:, :1] * 3) % 7], axis=1)
    lab = ((Y[:, 0] // 4 + Y[:, 1] // 3) % 4).astype(np.int64)
    out["lattice_400_ties"] = (X, Y, lab, 200, (8, 30), False)
    # small: trust/continuity and a short k_max
    rng = np.random.default_rng(34)
    X = rng.standard_normal((40, 5))
    Y = rng.standard_normal((40, 2))
    out["tiny_40"] = (X, Y, None, 7, (10,), False)
    return out


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    from ivhd import metrics

    arrays = {}
    for name, (X, Y, lab, k_max, ks, pre) in curve_inputs().items():
        cur = metrics.evaluate_embedding(X, Y, labels=lab, k_max=k_max, nn_max=20, report_ks=ks,
                                         x_precomputed=pre)
        arrays[f"{name}/q_nx"] = cur.q_nx
        arrays[f"{name}/r_nx"] = cur.r_nx
        arrays[f"{name}/auc_rnx"] = np.float64(cur.auc_rnx)
        if lab is not None:
            arrays[f"{name}/g_nn"] = cur.g_nn
            arrays[f"{name}/auc_gnn"] = np.float64(cur.auc_gnn)
        arrays[f"{name}/trust"] = np.array([cur.trust[k] for k in ks if k < len(Y) / 2])
        arrays[f"{name}/continuity"] = np.array([cur.continuity[k] for k in ks if k < len(Y) / 2])
        if not pre:
            _, _, _, auc = metrics.rnx_curve(X, Y, k_max=k_max)
            arrays[f"{name}/rnx_auc_direct"] = np.float64(auc)
            t, c = metrics.trust_continuity(X, Y, ks[0])
            arrays[f"{name}/tc_direct"] = np.array([t, c])
        if not pre:
            (dl, ds), (rho, rr), r2 = metrics.shepard_and_corank(X, Y, sample_pairs=min(3000, len(Y) * 4), seed=3)
            arrays[f"{name}/shepard_rho"] = rho
            arrays[f"{name}/shepard_r"] = rr
            arrays[f"{name}/shepard_r2"] = np.float64(r2)
            arrays[f"{name}/shepard_deltas"] = dl
        print(name, X.shape, cur.summary())
    np.savez_compressed(OUT, **arrays)


if __name__ == "__main__":
    main()
