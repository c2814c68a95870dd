mkdir -p gpurun_out
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "c3 rc=$?"
for w in c1 c2-adadelta c2-nesterov c4; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-knn > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"
done
timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 --no-knn --no-cpu > gpurun_out/c5.json 2> gpurun_out/c5.err; echo "c5 rc=$?"
for f in gpurun_out/ref.json gpurun_out/bench.json gpurun_out/bench_c*.json gpurun_out/c5.json; do python -c "
import json,sys; d=json.load(open('$f')); e=d.get('e2e') or {}; print('$f', d.get('value'), e.get('value'), e.get('s_per_embed'), d.get('ms_per_step'))"; done
