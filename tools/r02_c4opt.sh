#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_c4opt.txt
: > $O
for rep in 1 2; do
for a in "16,32" "16,32,fuse_shadow=1" "16,32,g:tc_narrow_max_tiles=65" "16,32,node_prio=1" "16,32,node_prio=1,prio_levels=3" "20,40" "24,48" "12,36"; do
  echo -n "$a " >> $O
  timeout 300 python tools/c4_bench.py $a >> $O 2>&1
done
done
