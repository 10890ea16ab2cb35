#!/bin/bash
# quick GPU pass: gpu tests, critical path at two sizes, short bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/critpath.py --n 16384 > gpurun_out/crit16384.txt 2>&1
timeout 600 python tools/critpath.py --n 65536 > gpurun_out/crit65536.txt 2>&1
