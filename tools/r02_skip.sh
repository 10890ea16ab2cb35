#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_skip.txt
timeout 1200 python tools/opt_sweep.py --n 65536 --reps 3 --set "" --set dev_skip=2 --set dev_skip=9 --set dev_skip=4194304 --set dev_skip=25166400 --set dev_skip=32 --set dev_skip=65536 --set dev_skip=11 > $O 2>&1
timeout 600 python tools/opt_sweep.py --n 16384 --reps 5 --set "" --set dev_skip=2 --set dev_skip=9 --set dev_skip=4194304 --set dev_skip=25166400 --set dev_skip=65536 >> $O 2>&1
