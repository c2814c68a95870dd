#!/bin/bash
# One call on an N-GPU box (profiles/r02_multigpu_recipe.md): the sharded GPU
# tests, then bench lines at 1/2/4/8 ranks (or up to the GPUs present) for the
# C3, C4 and C5 workloads through the fused P2P exchange, NVLink counters around
# the C4 run.  Outputs under gpurun_out/mgpu_*.
set -u
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
echo "GPUs: $NG" > gpurun_out/mgpu_summary.txt
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_system.py -q -m gpu -k "sharded or distributed or peer" \
  > gpurun_out/mgpu_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/mgpu_summary.txt
port=29611
for w in c3 c4 c5; do
  for n in 1 2 4 8; do
    [ "$n" -gt "$NG" ] && continue
    port=$((port + 1))
    extra="--no-knn"; [ "$w" != c3 ] && extra="--no-knn --no-cpu"
    [ "$w" = c4 ] && [ "$n" = "$NG" ] && nvidia-smi nvlink -gt d > gpurun_out/mgpu_nvl_before.txt 2>&1
    if [ "$n" = 1 ]; then
      timeout 1800 python bench.py --workload $w --steps 3 --warmup 3 $extra > gpurun_out/mgpu_${w}_$n.json 2> gpurun_out/mgpu_${w}_$n.err
    else
      timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $port bench.py --gpus $n --workload $w --steps 3 --warmup 3 $extra \
        > gpurun_out/mgpu_${w}_$n.json 2> gpurun_out/mgpu_${w}_$n.err
    fi
    rc=$?
    [ "$w" = c4 ] && [ "$n" = "$NG" ] && nvidia-smi nvlink -gt d > gpurun_out/mgpu_nvl_after.txt 2>&1
    python - "$w" "$n" "$rc" >> gpurun_out/mgpu_summary.txt <<'PY'
import json, sys
w, n, rc = sys.argv[1:]
try:
    d = json.loads([l for l in open(f"gpurun_out/mgpu_{w}_{n}.json") if l.startswith("{")][-1])
    nv = d.get("nvlink") or {}
    print(w, n, "rc", rc, "value %.4g" % d["value"], "ms/step %.2f" % d["ms_per_step"], "e2e", (d.get("e2e") or {}).get("value"),
          "nvlink GB/s", nv.get("achieved_gbs"))
except Exception as e:
    print(w, n, "rc", rc, "no line:", e)
PY
  done
done
cat gpurun_out/mgpu_summary.txt
