#!/bin/bash
# every bench line of the round (one GPU), into gpurun_out/r02_bench_*.json
mkdir -p gpurun_out
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference_c3.json 2> gpurun_out/r02_ref.err; echo "ref rc=$?"
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_c3.err; echo "c3 rc=$?"
for w in c1 c2-adadelta c2-nesterov c4; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-knn > gpurun_out/r02_bench_$w.json 2> gpurun_out/r02_$w.err; echo "$w rc=$?"
done
timeout 1200 python bench.py --workload c5 --steps 2 --warmup 3 --no-knn --no-cpu > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_c5.err; echo "c5 rc=$?"
for f in gpurun_out/r02_bench_*.json; do python -c "
import json,sys
d=json.load(open('$f')); e=d.get('e2e') or {}; r=d.get('roofline') or {}
print('$f', 'value %.4g' % d['value'], 'ms/step %.2f' % d['ms_per_step'], 'e2e %s' % e.get('value'), 'frac %s' % r.get('frac'))"; done
