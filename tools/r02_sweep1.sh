#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_sweep1.txt
timeout 900 python tools/opt_sweep.py --n 65536 --set shadow_per_block=0 --set "" --set syrk_split_min=16384 --set syrk_split_min=8192 --set syrk_split_min=4096 --set shadow_per_block=0,syrk_split_min=16384 > $O 2>&1
timeout 600 python tools/opt_sweep.py --n 16384 --reps 9 --set shadow_per_block=0 --set "" --set syrk_split_min=8192 --set syrk_split_min=2048 --set syrk_split_min=1024 >> $O 2>&1
timeout 600 python tools/critpath.py --n 16384 --json gpurun_out/r02_crit16384_spb.json > gpurun_out/r02_crit16384_spb.txt 2>&1
timeout 600 python tools/critpath.py --n 65536 --json gpurun_out/r02_crit65536_spb.json > gpurun_out/r02_crit65536_spb.txt 2>&1
timeout 600 python tools/c4_bench.py 16,32 >> $O 2>&1
