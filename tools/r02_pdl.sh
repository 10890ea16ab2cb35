#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_pdl.txt
timeout 300 python tools/check_rn.py > $O 2>&1
timeout 300 python tools/potrf_clk.py >> $O 2>&1
timeout 300 python tools/opt_sweep.py --n 16384 --reps 9 --set use_pdl=0 --set "" >> $O 2>&1
timeout 600 python tools/opt_sweep.py --n 65536 --reps 4 --set use_pdl=0 --set "" >> $O 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r02_pytest_pdl.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_pdl.log
timeout 600 python tools/c4_bench.py 16,32,use_pdl=0 16,32 >> $O 2>&1
