#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_sweep3.txt
timeout 1500 python tools/opt_sweep.py --n 65536 --reps 4 --set "" --set trsm_row_split_min=8192,syrk_split_min=8192 --set trsm_row_split_min=16384,syrk_split_min=16384,lookahead_prio=0 --set mma32w_max_log2=26 --set bulk_tiles_per_cta=2 > $O 2>&1
timeout 1200 python tools/c4_bench.py 16,32 16,32,mma32w_max_log2=26 16,32,mma32w_max_log2=25 20,40 12,24 >> $O 2>&1
