#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_sweep2.txt
timeout 900 python tools/opt_sweep.py --n 16384 --reps 9 --set "" --set sub32_max_rows=256 --set sub32_max_rows=1024 --set sub32_max_rows=4096 --set sub32_max_rows=256,syrk_split_min=1024 --set sub32_max_rows=4096,syrk_split_min=512 > $O 2>&1
timeout 900 python tools/opt_sweep.py --n 65536 --reps 4 --set "" --set sub32_max_rows=256 --set sub32_max_rows=4096 --set sub32_max_rows=4096,syrk_split_min=16384 >> $O 2>&1
timeout 600 python tools/critpath.py --n 16384 --opt sub32_max_rows=4096 --json gpurun_out/r02_crit16384_sub.json > gpurun_out/r02_crit16384_sub.txt 2>&1
timeout 900 python tools/critpath.py --n 65536 --opt sub32_max_rows=4096 --json gpurun_out/r02_crit65536_sub.json > gpurun_out/r02_crit65536_sub.txt 2>&1
timeout 300 python tools/gemm_stamps.py > gpurun_out/r02_gemm_stamps.txt 2>&1
timeout 600 python tools/c4_bench.py 16,32 >> $O 2>&1
