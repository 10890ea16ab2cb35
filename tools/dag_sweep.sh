#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/dag.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for s in 0 8192 4096 2048 1024 512; do
 for d in 1 0; do
  echo "split=$s dag=$d" >> gpurun_out/dag.txt
  timeout 300 python tools/critpath.py --n 65536 --opt syrk_split_min=$s --opt dag_graph=$d | head -1 | cut -c1-200 >> gpurun_out/dag.txt 2>&1
  timeout 300 python tools/critpath.py --n 16384 --opt syrk_split_min=$s --opt dag_graph=$d | head -1 | cut -c1-200 >> gpurun_out/dag.txt 2>&1
 done
done
