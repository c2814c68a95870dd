L=paper_2303_05455_b200/libivhd_b200.so
python tools/kernel_sweep.py --graphs mixture:1400000 $L $L@IVHD_LPT_C0=0 $L@IVHD_LPT_C0=1 $L@IVHD_LPT_C0=6 $L@IVHD_LPT_C0=12 $L@IVHD_CARVEOUT=50 $L@IVHD_CARVEOUT=25 > gpurun_out/c0_sweep.txt 2>&1; cat gpurun_out/c0_sweep.txt
