#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_look.txt
timeout 900 python -m pytest tests -x -q -m gpu -k "lookahead or factor_matches or c2" > gpurun_out/r02_pytest_look.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_look.log
timeout 1500 python tools/opt_sweep.py --n 65536 --reps 4 --set "" --set trsm_row_split_min=8192,syrk_split_min=8192 --set trsm_row_split_min=8192,syrk_split_min=8192,lookahead_prio=0 --set trsm_row_split_min=16384,syrk_split_min=16384 --set trsm_row_split_min=4096,syrk_split_min=4096 --set trsm_row_split_min=2048,syrk_split_min=2048 > $O 2>&1
timeout 600 python tools/opt_sweep.py --n 16384 --reps 7 --set "" --set trsm_row_split_min=2048,syrk_split_min=2048 --set trsm_row_split_min=4096,syrk_split_min=4096 --set trsm_row_split_min=1024,syrk_split_min=1024 >> $O 2>&1
timeout 900 python tools/c4_bench.py 16,32 16,32,trsm_row_split_min=2048,syrk_split_min=2048 16,32,trsm_row_split_min=4096,syrk_split_min=4096 >> $O 2>&1
