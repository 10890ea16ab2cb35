#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/sched2.txt
for s in 0 1024; do for t in 0 1; do for m in 0 136; do
  echo "split=$s tiles=$t maxcta=$m" >> gpurun_out/sched2.txt
  timeout 300 python tools/critpath.py --n 65536 --opt syrk_split_min=$s --opt bulk_tiles_per_cta=$t --opt bulk_max_ctas=$m | head -1 | grep -o 'graph_ms": [0-9.]*' >> gpurun_out/sched2.txt 2>&1
  timeout 300 python tools/critpath.py --n 16384 --opt syrk_split_min=$s --opt bulk_tiles_per_cta=$t --opt bulk_max_ctas=$m | head -1 | grep -o 'graph_ms": [0-9.]*' >> gpurun_out/sched2.txt 2>&1
done; done; done
