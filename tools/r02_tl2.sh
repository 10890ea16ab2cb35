#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_tl2.txt
: > $O
timeout 300 python tools/timeline_bins.py --n 65536 --bin 4 --opt trsm_row_split_min=4096 --opt syrk_split_min=4096 >> $O 2>&1
timeout 300 python tools/timeline_bins.py --n 65536 --bin 4 --opt syrk_split_min=4096 >> $O 2>&1
