#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_res.txt
L=trsm_row_split_min=8192,syrk_split_min=8192
timeout 1800 python tools/opt_sweep.py --n 65536 --reps 3 --set "" --set bulk_tiles_per_cta=0,bulk_max_ctas=140 --set bulk_tiles_per_cta=0,bulk_max_ctas=132 --set bulk_tiles_per_cta=0,bulk_max_ctas=120 --set bulk_tiles_per_cta=0,bulk_max_ctas=140,$L --set bulk_tiles_per_cta=0,bulk_max_ctas=132,$L --set bulk_tiles_per_cta=0,bulk_max_ctas=120,$L > $O 2>&1
timeout 600 python tools/opt_sweep.py --n 16384 --reps 7 --set "" --set bulk_tiles_per_cta=0,bulk_max_ctas=140 --set bulk_tiles_per_cta=0,bulk_max_ctas=128 >> $O 2>&1
