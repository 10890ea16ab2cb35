#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_conn3.txt
: > $O
for c in 8 32; do
  echo "conn=$c" >> $O
  CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 600 python tools/opt_sweep.py --n 65536 --reps 4 --set "" --set trsm_row_split_min=4096,syrk_split_min=4096 >> $O 2>&1
  CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 300 python tools/opt_sweep.py --n 16384 --reps 4 --set "" --set trsm_row_split_min=2048,syrk_split_min=2048 >> $O 2>&1
done
