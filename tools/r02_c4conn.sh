#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_c4conn.txt
: > $O
for i in 1 2 3 4 5; do
  for c in default 32; do
    if [ $c = default ]; then
      echo -n "conn=default " >> $O; TC_PAIR_MIN=512 timeout 300 python tools/c4_bench.py 16,32 >> $O 2>&1
    else
      echo -n "conn=$c " >> $O; CUDA_DEVICE_MAX_CONNECTIONS=$c TC_PAIR_MIN=512 timeout 300 python tools/c4_bench.py 16,32 >> $O 2>&1
    fi
  done
done
