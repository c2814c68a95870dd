#!/bin/bash
# quick GPU loop: parity tests + short bench + launch list (used via gpurun)
set -o pipefail
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -${TAIL:-15}
python bench.py --steps 3 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
