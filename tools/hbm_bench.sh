#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python tools/critpath.py --n 65536 > gpurun_out/crit65536.txt 2>&1
timeout 300 python tools/gemm_bench.py simt_f64 > gpurun_out/gemm_f64.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:k_export|k_import|k_quant1|k_shadow" --csv --log-file gpurun_out/hbm.csv python tools/critpath.py --n 65536 --profile-only > gpurun_out/hbm.log 2>&1
