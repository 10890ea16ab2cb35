#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_base2.txt
timeout 600 python tools/potrf_clk.py > $O 2>&1
timeout 600 python tools/opt_sweep.py --n 16384 --reps 9 --set "" --set syrk_split_min=512 --set syrk_split_min=1024 >> $O 2>&1
timeout 900 python tools/opt_sweep.py --n 65536 --reps 4 --set "" --set syrk_split_min=512 >> $O 2>&1
timeout 600 python tools/c4_bench.py 16,32 16,32,syrk_split_min=512 >> $O 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench2.jsonl 2> gpurun_out/r02_bench2.err
