#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_c4c3.txt
: > $O
for i in 1 2; do
  timeout 600 python tools/c4_after_c3.py >> $O 2>&1
  timeout 600 python tools/c4_after_c3.py c3 >> $O 2>&1
done
