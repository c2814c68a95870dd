"""Generate the golden fixtures in this directory from the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package `ivhd` from /root/reference/pkg/src, drives
its public functions (ConnectionSet/compute_forces/stress, the optimizers,
_Run + the loop body of run_embedding, run_embedding itself) on small seeded
inputs and stores inputs and outputs as .npz files.  The fixtures pin the
oracle (tests/test_oracle_golden.py) and, on the GPU box, the CUDA path
(tests/test_gpu_parity.py) — neither test reads /root/reference at run time.
"""

import json
import os
import sys
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import ivhd  # noqa: F401
    from ivhd import engine, forces, knng, optim

    return engine, forces, knng, optim


def blob_data():
    # same recipe as the reference's test_engine.py:17-22 fixture
    rng = np.random.default_rng(0)
    centers = rng.standard_normal((4, 8)) * 4
    return np.vstack([centers[i] + rng.standard_normal((50, 8)) for i in range(4)])


def random_conn_arrays(m, nn, rn, rng, mode):
    # same construction as the reference's test_forces.py:16-30 helper
    rows = []
    for i in range(m):
        others = rng.choice([j for j in range(m) if j != i], size=nn + rn, replace=False)
        rows += [(i, int(j), False) for j in others[:nn]]
        rows += [(i, int(j), True) for j in others[nn:]]
    edges = np.array([(i, j) for i, j, _ in rows], dtype=np.int32)
    is_rn = np.array([r for _, _, r in rows])
    targets = np.where(is_rn, 1.0, 0.0) if mode == "binary" else rng.uniform(0.2, 1.5, len(edges))
    return edges, targets, is_rn


def make_force_cases(F):
    cases = {}
    rng = np.random.default_rng(1234)
    k = 0
    for m, nn, rn in ((30, 3, 2), (200, 3, 1), (500, 2, 1)):
        for mode in ("binary", "euclidean"):
            for norm in ("l2", "l1"):
                for scaled in (False, True):
                    edges, targets, is_rn = random_conn_arrays(m, nn, rn, rng, mode)
                    scale = rng.uniform(0.5, 2.0, len(edges)) if scaled else None
                    conn = F.ConnectionSet(edges, targets, is_rn, scale=scale)
                    for dim in (2, 3):
                        Y = rng.uniform(-1, 1, (m, dim))
                        c = float(rng.choice([0.01, 0.1, 0.5]))
                        f, e = F.compute_forces(Y, conn, c, norm, with_stress=True)
                        s = F.stress(Y, conn, c, norm)
                        p = f"c{k}_"
                        cases.update({
                            p + "edges": edges, p + "targets": targets, p + "is_random": is_rn,
                            p + "scale": np.zeros(0) if scale is None else scale,
                            p + "Y": Y, p + "c": np.array(c), p + "norm": np.array(norm),
                            p + "force": f, p + "stress_with": np.array(e),
                            p + "stress": np.array(s),
                        })
                        k += 1
    cases["n_cases"] = np.array(k)
    np.savez_compressed(os.path.join(HERE, "force_cases.npz"), **cases)
    print("force_cases:", k)


def replay(engine, F, optim, graph, cfg, steps):
    """Step-by-step replay of run_embedding's loop body (engine.py:346-384)."""
    run = engine._Run(graph, cfg)
    out = {"Y0": run.positions.copy(), "rn": run.rn_assignments.copy()}
    forces, positions, stresses, bs = [], [], [], []
    for it in range(steps):
        conn = run.conn_full
        ev = run.optimizer.lookahead(run.positions)
        if ev is run.positions:
            f, e = F.compute_forces(ev, conn, run.c, "l2", rng=run.rng, with_stress=True)
        else:
            f = F.compute_forces(ev, conn, run.c, "l2", rng=run.rng)
            e = F.stress(run.positions, conn, run.c, "l2")
        new = optim.step_optimizer(run.optimizer, run.positions, f)
        run.positions = new
        forces.append(f)
        positions.append(new.copy())
        stresses.append(e)
        bs.append(run.optimizer.step_size)
    out.update(force=np.array(forces), positions=np.array(positions),
               stress=np.array(stresses), b=np.array(bs))
    return out


def make_replays(engine, F, optim, knng):
    data = blob_data()
    graph = knng.build_exact_knn(data, 12)
    blob = {"data": data, "neighbors": graph.neighbors, "distances": graph.distances}
    np.savez_compressed(os.path.join(HERE, "blob_graph.npz"), **blob)
    meta = {}
    for kind in ("force-directed", "sgd", "momentum", "nesterov", "adam", "adadelta"):
        for dim in (2, 3):
            cfg = engine.EmbeddingConfig(nn=3, rn=1, c=0.1, iterations=10, seed=7,
                                         optimizer=kind, target_dim=dim)
            r = replay(engine, F, optim, graph, cfg, 10)
            name = f"replay_{kind}_d{dim}"
            np.savez_compressed(os.path.join(HERE, name + ".npz"), **r)
            meta[name] = {"nn": 3, "rn": 1, "c": 0.1, "seed": 7, "optimizer": kind,
                          "target_dim": dim, "steps": 10}
    return graph, data, meta


def make_runs(engine, knng, graph, data, meta):
    from ivhd.datasets import Dataset
    from ivhd.errors import NumericalDivergenceError
    from ivhd.optim import IntegratorParams

    runs = {
        "fd_300": dict(nn=3, rn=1, c=0.1, iterations=300, seed=3),
        "fd_c005_400": dict(nn=3, rn=1, c=0.05, iterations=400, seed=5),
        "nesterov_200": dict(nn=3, rn=1, c=0.1, iterations=200, seed=2, optimizer="nesterov"),
        "adadelta_200": dict(nn=3, rn=1, c=0.1, iterations=200, seed=2, optimizer="adadelta"),
        "adam_200": dict(nn=3, rn=1, c=0.1, iterations=200, seed=2, optimizer="adam"),
        "phased_rnn_l1": dict(nn=3, rn=1, c=0.1, iterations=120, seed=6,
                              rnn_final_steps=40, l1_final_steps=15),
        "resample_p7": dict(nn=3, rn=1, c=0.1, iterations=60, seed=8, rn_resample_period=7),
        "rollback_tau": dict(nn=3, rn=1, c=0.1, iterations=40, seed=9,
                             integrator={"tau": 0.05, "b": 0.01}),
        "no_adapt": dict(nn=3, rn=1, c=0.1, iterations=50, seed=10,
                         integrator={"a": 0.9, "b": 0.003, "auto_adapt": False}),
        "euclid_60": dict(nn=3, rn=1, c=0.1, iterations=60, seed=4, distance_mode="euclidean"),
        "dim3_40": dict(nn=2, rn=1, c=0.1, iterations=40, seed=2, target_dim=3),
        "zero_iter": dict(nn=3, rn=1, c=0.1, iterations=0, seed=11),
    }
    for name, kw in runs.items():
        cfg = engine.EmbeddingConfig(**kw)
        ds = Dataset(data) if kw.get("distance_mode") == "euclidean" else None
        res = engine.run_embedding(graph=graph, config=cfg, dataset=ds)
        np.savez_compressed(
            os.path.join(HERE, f"run_{name}.npz"),
            points=res.embedding.points, stress=np.array(res.trace.stress),
            b=np.array(res.trace.step_size), final_stress=np.array(res.state.stress),
            deltas=res.state.deltas, rn=res.state.rn_assignments,
            iteration=np.array(res.state.iteration),
        )
        meta[f"run_{name}"] = kw
    # divergence (test_engine.py:114-122)
    kw = dict(nn=3, rn=1, c=0.1, iterations=500, seed=1,
              integrator={"a": 1.0, "b": 1e6, "auto_adapt": False})
    try:
        engine.run_embedding(graph=graph, config=engine.EmbeddingConfig(
            **{**kw, "integrator": IntegratorParams(**kw["integrator"])}))
        raise RuntimeError("expected divergence")
    except NumericalDivergenceError as err:
        np.savez_compressed(os.path.join(HERE, "run_diverge.npz"),
                            iteration=np.array(err.iteration),
                            positions=err.state.positions, stress=np.array(err.state.stress))
    meta["run_diverge"] = kw


def main():
    warnings.simplefilter("ignore")
    engine, F, knng, optim = _import_reference()
    make_force_cases(F)
    graph, data, meta = make_replays(engine, F, optim, knng)
    make_runs(engine, knng, graph, data, meta)
    with open(os.path.join(HERE, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(meta), "fixtures")


if __name__ == "__main__":
    main()
