#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/mma_sweep.txt
for v in -1 24 26 29; do
  echo "mma32_max_log2=$v" >> gpurun_out/mma_sweep.txt
  for rep in 1 2; do
  timeout 300 python tools/critpath.py --n 65536 --opt mma32_max_log2=$v | head -1 | grep -o 'graph_ms": [0-9.]*' >> gpurun_out/mma_sweep.txt
  timeout 300 python tools/critpath.py --n 16384 --opt mma32_max_log2=$v | head -1 | grep -o 'graph_ms": [0-9.]*' >> gpurun_out/mma_sweep.txt
  done
done
