#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/fp64_peak.py gpurun_out/r02_fp64_peak.json > gpurun_out/r02_fp64_peak.log 2>&1
timeout 600 python tools/gemm_ops.py 65536 > gpurun_out/r02_gemm_ops_65536.txt 2>&1
timeout 300 python tools/gemm_ops.py 16384 > gpurun_out/r02_gemm_ops_16384.txt 2>&1
timeout 600 python tools/critpath.py --n 65536 --json gpurun_out/r02_crit65536.json > gpurun_out/r02_crit65536b.txt 2>&1
timeout 300 python tools/critpath.py --n 16384 --json gpurun_out/r02_crit16384.json > gpurun_out/r02_crit16384b.txt 2>&1
timeout 600 python -m pytest tests -x -q -m gpu -k "factor or potrf or c1 or c2" > gpurun_out/r02_pytest_sub.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_sub.log
