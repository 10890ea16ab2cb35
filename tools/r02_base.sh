#!/bin/bash
# round-2 baseline pass: gpu tests, default bench line, critical paths
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -q -d CLOCK,POWER | head -60 > gpurun_out/r02_smi.txt
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r02_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02_bench.jsonl 2> gpurun_out/r02_bench.err; echo "rc=$?" >> gpurun_out/r02_bench.err
timeout 300 python tools/critpath.py --n 16384 > gpurun_out/r02_crit16384.txt 2>&1
timeout 600 python tools/critpath.py --n 65536 > gpurun_out/r02_crit65536.txt 2>&1
