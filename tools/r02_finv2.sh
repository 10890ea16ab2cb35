#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_finv2.txt
timeout 300 python tools/potrf_clk.py > $O 2>&1
timeout 600 python tools/opt_sweep.py --n 16384 --reps 9 --set fuse_inverse=0 --set "" >> $O 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "factor_matches or inverse or c2" > gpurun_out/r02_pytest_finv2.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_finv2.log
