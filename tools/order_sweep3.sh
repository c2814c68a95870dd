L=paper_2303_05455_b200/libivhd_b200.so
python tools/kernel_sweep.py --graphs planted:100000000,planted:10000000 $L $L@IVHD_ORDER_WINDOW=1 $L@IVHD_ORDER_WINDOW=64 $L@IVHD_ORDER_WINDOW=256 $L@IVHD_ORDER_WINDOW=8192 > gpurun_out/order_sweep3.txt 2>&1; cat gpurun_out/order_sweep3.txt
