#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_rn2.txt
timeout 300 python tools/check_rn.py > $O 2>&1
timeout 300 python tools/potrf_clk.py >> $O 2>&1
timeout 300 python tools/opt_sweep.py --n 16384 --reps 9 --set "" --set use_pdl=1 >> $O 2>&1
