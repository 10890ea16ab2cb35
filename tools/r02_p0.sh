#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_p0.txt
timeout 300 python tools/gemm_stamps.py > $O 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "factor or kernels or gemm or c2" > gpurun_out/r02_pytest_p0.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_p0.log
timeout 300 python tools/opt_sweep.py --n 16384 --reps 9 --set "" >> $O 2>&1
timeout 600 python tools/opt_sweep.py --n 65536 --reps 4 --set "" >> $O 2>&1
timeout 600 python tools/c4_bench.py 16,32 >> $O 2>&1
timeout 600 python tools/gemm_ops.py 65536 > gpurun_out/r02_gemm_ops_65536b.txt 2>&1
