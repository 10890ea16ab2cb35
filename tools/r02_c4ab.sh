#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_c4ab.txt
: > $O
for i in 1 2; do
timeout 600 python tools/c4_bench.py 16,32,fuse_shadow=0 >> $O 2>&1
timeout 600 python tools/c4_bench.py 16,32 >> $O 2>&1
done
