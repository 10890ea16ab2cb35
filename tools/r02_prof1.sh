#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "factor or host or export or c2 or c1" > gpurun_out/r02_pytest_exp.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_exp.log
timeout 600 python tools/opt_sweep.py --n 65536 --reps 4 --set "" --set dev_skip=2 > gpurun_out/r02_export.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches16384.csv python tools/critpath.py --n 16384 --profile-only > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_potrf_v2 -s 5 -c 1 -o gpurun_out/r02_potrf python tools/critpath.py --n 16384 --profile-only > gpurun_out/r02_potrf_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leaf_inv2 -s 5 -c 1 -o gpurun_out/r02_inv python tools/critpath.py --n 16384 --profile-only > gpurun_out/r02_inv_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_export -s 20 -c 2 -o gpurun_out/r02_export python tools/critpath.py --n 16384 --profile-only > gpurun_out/r02_export_ncu.log 2>&1
timeout 300 python tools/launch_rate.py > gpurun_out/r02_launch_rate.txt 2>&1
