"""TEST INFRASTRUCTURE ONLY — CPU oracle for the IVHD embedding loop.

This package restates, in numpy, the reference algorithm for the one hot path
this repository accelerates (the IVHD embedding loop of arXiv 2303.05455 as
implemented by the reference package `ivhd`, `pkg/src/ivhd/engine.py:312-414`,
`forces.py:78-186`, `optim.py:80-263`).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may
import it, and only as the checker / the timed CPU baseline — never as the
product path.  The product (`paper_2303_05455_b200`) runs on the CUDA library
and fails loudly when it is missing.

Parity pinning: the oracle is checked against golden vectors produced by the
reference itself (imported in the build container from /root/reference) —
see `tests/golden/make_golden.py` and `tests/test_oracle_golden.py`.
"""

from .ivhd_oracle import (  # noqa: F401
    Connections,
    OracleRun,
    accumulate,
    build_connections,
    components,
    csr_forces,
    curve_pass,
    forces,
    init_layout,
    make_state,
    optimizer_step,
    rnn_keep_mask,
    sample_rn,
    stress,
    symmetrise,
)
