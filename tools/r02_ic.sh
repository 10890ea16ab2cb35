#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_ic.txt
: > $O
timeout 1700 python tools/opt_sweep.py --n 65536 --reps 4 --set "" --set startup_order=1,import_chain=8 --set startup_order=1,import_chain=32 --set import_chain=16 --set "" --set startup_order=1,import_chain=8 >> $O 2>&1
timeout 400 python tools/opt_sweep.py --n 16384 --reps 4 --set "" --set startup_order=1,import_chain=8 >> $O 2>&1
timeout 300 python tools/trace_bins.py --n 65536 --opt startup_order=1 --opt import_chain=8 --json gpurun_out/tr9.json > /dev/null 2>&1
