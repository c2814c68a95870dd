#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
L=paper_2303_05455_b200/libivhd_b200.so
python tools/kernel_sweep.py --graphs planted:100000000,planted:10000000,planted:30000000 $L $L@IVHD_CONTIG=0 > gpurun_out/contig_sweep.txt 2>&1; cat gpurun_out/contig_sweep.txt
bash tools/c5_ncu.sh
