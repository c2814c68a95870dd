"""Route the reference package's own callers through the B200 path.

The reference's CLI (`ivhd embed`, cli.py:227; kNN at cli.py:102; metrics at
cli.py:283/298) and steering server (`SteerServer._drive`, server.py:76) bind
`run_embedding`, `knng.build_exact_knn` and the metrics by module attribute.
`install()` re-points those attributes (and the operators
`forces.compute_forces` / `forces.stress`, forces.py:78,139) at this package,
so the unmodified callers run on the GPU; `uninstall()` puts the originals
back.  This is the shim INTEGRATION.md §2 describes, shipped as a function:

    import ivhd, paper_2303_05455_b200.reference_shim as shim
    shim.install(ivhd)          # e.g. from ivhd/__init__.py when IVHD_BACKEND=b200

Nothing here computes; the replaced functions keep the reference's signatures,
result types and exception classes (see INTEGRATION.md for the documented
limits of the GPU metrics).
"""

import importlib

# (reference module, attribute) -> (this package's module, attribute)
_ROUTES = (
    ("engine", "run_embedding", "", "run_embedding"),
    ("cli", "run_embedding", "", "run_embedding"),
    ("server", "run_embedding", "", "run_embedding"),
    ("forces", "compute_forces", "", "compute_forces"),
    ("forces", "stress", "", "stress"),
    ("knng", "build_exact_knn", ".knng", "build_exact_knn"),
    ("metrics", "neighbor_hit", ".metrics", "neighbor_hit"),
    ("metrics", "rnx_curve", ".metrics", "rnx_curve"),
    ("metrics", "gnn_curve", ".metrics", "gnn_curve"),
    ("metrics", "trust_continuity", ".metrics", "trust_continuity"),
    ("metrics", "evaluate_embedding", ".metrics", "evaluate_embedding"),
    ("metrics", "shepard_and_corank", ".metrics", "shepard_and_corank"),
    ("metrics", "compute_ranks", ".metrics", "compute_ranks"),
    ("metrics", "RankData", ".metrics", "RankData"),
    ("metrics", "MetricCurves", ".metrics", "MetricCurves"),
)


def _ours(mod, name):
    m = importlib.import_module("paper_2303_05455_b200" + mod)
    return getattr(m, name)


def install(ivhd=None, modules=("engine", "cli", "server", "forces", "knng", "metrics")):
    """Re-point the reference modules' attributes at this package.  `ivhd`:
    the reference package (imported if None).  Reference modules that cannot
    be imported (e.g. `server` without fastapi) are skipped.  Returns the
    replaced originals, {(module, attribute): object}, for `uninstall`."""
    if ivhd is None:
        ivhd = importlib.import_module("ivhd")
    saved = {}
    for ref_mod, attr, our_mod, our_attr in _ROUTES:
        if ref_mod not in modules:
            continue
        try:
            target = importlib.import_module(f"{ivhd.__name__}.{ref_mod}")
        except ImportError:
            continue
        if not hasattr(target, attr):
            continue
        saved[(target.__name__, attr)] = getattr(target, attr)
        setattr(target, attr, _ours(our_mod, our_attr))
    return saved


def uninstall(saved):
    """Restore what `install` replaced."""
    for (mod, attr), obj in saved.items():
        setattr(importlib.import_module(mod), attr, obj)
