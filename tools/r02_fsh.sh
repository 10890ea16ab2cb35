#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_fsh.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02_pytest_fsh.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_fsh.log
timeout 900 python tools/opt_sweep.py --n 65536 --reps 4 --set fuse_shadow=0 --set "" --set fuse_shadow=0 --set "" > $O 2>&1
timeout 600 python tools/opt_sweep.py --n 16384 --reps 9 --set fuse_shadow=0 --set "" >> $O 2>&1
timeout 900 python tools/c4_bench.py 16,32,fuse_shadow=0 16,32 >> $O 2>&1
