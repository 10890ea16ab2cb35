#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_mma.txt
timeout 1200 python tools/opt_sweep.py --n 65536 --reps 3 --set "" --set mma32_max_log2=25 --set mma32_max_log2=26 --set mma32_max_log2=27 --set mma32w_max_log2=26 > $O 2>&1
timeout 600 python tools/opt_sweep.py --n 16384 --reps 7 --set "" --set mma32_max_log2=25 --set mma32_max_log2=26 >> $O 2>&1
timeout 900 python tools/c4_bench.py 16,32 16,32,mma32_max_log2=25 16,32,mma32_max_log2=26 >> $O 2>&1
