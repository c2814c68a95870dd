L=paper_2303_05455_b200/libivhd_b200.so
python tools/kernel_sweep.py --graphs planted:100000000,planted:30000000 $L $L@IVHD_ORDER_WINDOW=256 $L@IVHD_ORDER_WINDOW=512 $L@IVHD_ORDER_WINDOW=1024 $L@identity@IVHD_LPT=0 > gpurun_out/order_sweep2.txt 2>&1
