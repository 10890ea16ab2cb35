#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/conn.txt
for c in 8 16 32; do
  echo "CUDA_DEVICE_MAX_CONNECTIONS=$c" >> gpurun_out/conn.txt
  CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 300 python tools/critpath.py --n 65536 --opt syrk_split_min=4096 | head -1 | cut -c1-200 >> gpurun_out/conn.txt 2>&1
  CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 300 python tools/critpath.py --n 16384 --opt syrk_split_min=4096 | head -1 | cut -c1-200 >> gpurun_out/conn.txt 2>&1
done
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 600 python tools/timeline.py --n 65536 --opt syrk_split_min=4096 > gpurun_out/timeline32.txt 2>&1
