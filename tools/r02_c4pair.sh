#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_c4pair.txt
: > $O
for i in 1 2 3; do
TC_PAIR_MIN=0 timeout 600 python tools/c4_bench.py 16,32 >> $O 2>&1
TC_PAIR_MIN=512 timeout 600 python tools/c4_bench.py 16,32 >> $O 2>&1
done
