#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_c4pair2.txt
: > $O
for rep in 1 2 3; do
for a in "16,32" "16,32,pair_min_tiles=512" "16,32,pair_min_tiles=1024"; do
  echo -n "$a " >> $O
  timeout 300 python tools/c4_bench.py $a >> $O 2>&1
done
done
