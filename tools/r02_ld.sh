#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_ld.txt
: > $O
timeout 300 python tools/potrf_clk.py >> $O 2>&1
timeout 400 python tools/opt_sweep.py --n 16384 --reps 4 --set "" >> $O 2>&1
timeout 900 python tools/opt_sweep.py --n 65536 --reps 4 --set "" >> $O 2>&1
timeout 900 python -m pytest tests -q -m gpu -x >> $O 2>&1
