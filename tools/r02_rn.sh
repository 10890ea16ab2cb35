#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/check_rn.py > gpurun_out/r02_rn.txt 2>&1
timeout 300 python tools/potrf_clk.py >> gpurun_out/r02_rn.txt 2>&1
timeout 300 python tools/opt_sweep.py --n 16384 --reps 7 --set "" >> gpurun_out/r02_rn.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "factor or c1 or c2 or potrs or batch" > gpurun_out/r02_pytest_rn.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_rn.log
