#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_c4opt2.txt
: > $O
for rep in 1 2; do
for a in "16,32" "16,32,bulk_tiles_per_cta=2" "16,32,bulk_tiles_per_cta=4" "16,32,bulk_tiles_per_cta=0" "16,32,crit_tiles_per_cta=1" "16,32,crit_tiles_per_cta=2" "16,32,fuse_shadow=0"; do
  echo -n "$a " >> $O
  timeout 300 python tools/c4_bench.py $a >> $O 2>&1
done
done
