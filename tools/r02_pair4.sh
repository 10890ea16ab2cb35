#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_pair4.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r02_pytest_pair4.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_pair4.log
timeout 900 python tools/opt_sweep.py --n 65536 --reps 4 --set g:tc_pair_min_tiles=0 --set "" --set g:tc_pair_min_tiles=0 --set "" > $O 2>&1
timeout 600 python tools/c4_bench.py 16,32 >> $O 2>&1
timeout 600 python tools/c4_bench.py 16,32 >> $O 2>&1
