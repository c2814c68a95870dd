#!/bin/bash
# refresh every bench line, then the ncu launch list and one full capture of the C3 step kernel
mkdir -p gpurun_out
bash tools/all_bench.sh
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --iterations 100 --no-e2e --no-cpu --no-knn > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 30 -c 1 -o gpurun_out/step_head -f \
  python bench.py --steps 1 --warmup 1 --iterations 100 --no-e2e --no-cpu --no-knn > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
