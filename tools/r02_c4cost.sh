#!/bin/bash
# C4 cost attribution: remove one class of kernels at a time (results garbage)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_c4cost.txt
: > $O
for ds in 0 3 65536 4194304 25166400 512 32 9 0; do
  echo -n "dev_skip=$ds " >> $O
  timeout 300 python tools/c4_bench.py 16,32,dev_skip=$ds >> $O 2>&1
done
