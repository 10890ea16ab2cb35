#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_f64.txt
timeout 300 python tools/leafclk.py > $O 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "factor or c1 or c2 or pure_f64 or textbook or ladder or blockops" > gpurun_out/r02_pytest_f64.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_f64.log
timeout 600 python tools/opt_sweep.py --n 8192 --cfg "[F16, F32, F64]" --reps 5 --set "" >> $O 2>&1
timeout 600 python tools/opt_sweep.py --n 1024 --b 128 --cfg "[F16, F64]" --reps 5 --set "" >> $O 2>&1
