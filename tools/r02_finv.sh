#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_finv.txt
timeout 1200 python -m pytest tests -x -q -m gpu -k "factor or inverse or c1 or c2 or c3 or lookahead or batch or potrs" > gpurun_out/r02_pytest_finv.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_finv.log
timeout 300 python tools/potrf_clk.py > $O 2>&1
timeout 600 python tools/opt_sweep.py --n 16384 --reps 9 --set fuse_inverse=0 --set "" >> $O 2>&1
timeout 900 python tools/opt_sweep.py --n 65536 --reps 4 --set fuse_inverse=0 --set "" >> $O 2>&1
timeout 900 python tools/c4_bench.py 16,32,fuse_inverse=0 16,32 >> $O 2>&1
