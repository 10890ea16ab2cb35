#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/potrf_clk.py > gpurun_out/r02_clk.txt 2>&1
timeout 300 python tools/opt_sweep.py --n 16384 --reps 7 --set "" >> gpurun_out/r02_clk.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_shadow --csv --log-file gpurun_out/r02_shadow.csv python tools/critpath.py --n 16384 --profile-only > /dev/null 2>&1
