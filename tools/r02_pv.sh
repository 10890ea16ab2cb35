#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_pv.txt
: > $O
timeout 300 python tools/potrf_clk.py >> $O 2>&1
timeout 600 python tools/opt_sweep.py --n 16384 --reps 4 --set "" >> $O 2>&1
timeout 900 python tools/opt_sweep.py --n 65536 --reps 4 --set "" >> $O 2>&1
timeout 900 python -m pytest tests/test_gpu_factor.py -q -x >> $O 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
timeout 900 $NCU -k regex:k_gemm_tc2ILi0E --launch-skip 87 -c 1 -o gpurun_out/r02z_gemm_tc2_top -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/r02z_f.log 2>&1
timeout 900 $NCU -k regex:k_gemm_tc2ILi0E --launch-skip 19 -c 1 -o gpurun_out/r02z_gemm_tc2_8192 -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/r02z_g.log 2>&1
