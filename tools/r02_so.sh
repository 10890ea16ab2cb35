#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_so.txt
: > $O
timeout 1500 python tools/opt_sweep.py --n 65536 --reps 4 --set "" --set startup_order=1 --set "" --set startup_order=1 >> $O 2>&1
timeout 400 python tools/opt_sweep.py --n 16384 --reps 4 --set "" --set startup_order=1 >> $O 2>&1
timeout 300 python tools/trace_bins.py --n 65536 --opt startup_order=1 --json gpurun_out/tr8.json > /dev/null 2>&1
