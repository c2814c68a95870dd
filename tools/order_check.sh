#!/bin/bash
# locality-driven vertex order: parity tests, then the kernel sweep and the C4/C5 bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
L=paper_2303_05455_b200/libivhd_b200.so
python tools/kernel_sweep.py --graphs planted:100000000,planted:10000000,mixture:1400000 $L > gpurun_out/order_auto.txt 2>&1; cat gpurun_out/order_auto.txt
timeout 600 python bench.py --workload c4 --steps 3 --warmup 3 --no-knn > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 --no-knn --no-cpu > gpurun_out/c5.json 2> gpurun_out/c5.err; echo "c5 rc=$?"
for f in gpurun_out/bench_c4.json gpurun_out/c5.json; do python -c "
import json; d=json.load(open('$f')); e=d.get('e2e') or {}; print('$f', d.get('value'), e.get('value'), e.get('s_per_embed'), d.get('ms_per_step'))"; done
