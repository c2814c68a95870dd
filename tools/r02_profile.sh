#!/bin/bash
# round-2 ncu evidence (one GPU): C3 step kernel in steady state (full set,
# warm L2), the bench launch list, and DRAM metrics of one C4 / C5 launch
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,lts__t_sectors.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
python tools/profile_c3.py 700 > gpurun_out/plain_c3.log 2>&1 && \
  ncu --set full --cache-control none --clock-control none --import-source on -k regex:step_kernel -s 600 -c 1 \
      -o gpurun_out/r02_c3_steady -f python tools/profile_c3.py 700 > gpurun_out/ncu_c3.log 2>&1; echo "c3 full rc=$?"
python bench.py --steps 1 --warmup 1 --iterations 200 --no-e2e --no-cpu --no-knn --no-quality > gpurun_out/plain_launch.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches_c3.csv \
      python bench.py --steps 1 --warmup 1 --iterations 200 --no-e2e --no-cpu --no-knn --no-quality > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
for w in c4 c5; do
  python bench.py --workload $w --iterations 6 --steps 1 --warmup 1 --no-e2e --no-cpu --no-knn > gpurun_out/plain_$w.log 2>&1 && \
    ncu --metrics $M --cache-control none --clock-control none -k regex:step_kernel -s 5 -c 1 --csv \
        python bench.py --workload $w --iterations 6 --steps 1 --warmup 1 --no-e2e --no-cpu --no-knn > gpurun_out/r02_${w}_ncu.csv 2> gpurun_out/r02_${w}_ncu.err; echo "$w rc=$?"
done
