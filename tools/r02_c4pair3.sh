#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_c4pair3.txt
: > $O
for rep in 1 2 3 4 5 6 7 8; do
  echo -n "16,32,pair_min_tiles=1024 " >> $O
  timeout 300 python tools/c4_bench.py 16,32,pair_min_tiles=1024 >> $O 2>&1
done
