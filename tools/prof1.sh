#!/bin/bash
# profiling pass: critical path, bench launch list, ncu full captures of the top kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/critpath.py --n 65536 --json gpurun_out/crit65536.json > gpurun_out/crit65536.txt 2>&1
timeout 300 python tools/critpath.py --n 16384 > gpurun_out/crit16384.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
   python bench.py --steps 1 --warmup 0 --e2e-steps 0 --cpu-n 0 > gpurun_out/bench_ncu.log 2>&1
IDX=$(python tools/critpath.py --n 65536 --ncu-pick)
echo "tc pick $IDX" > gpurun_out/ncu_pick.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc --launch-skip $IDX -c 1 \
   -o gpurun_out/ncu_gemm_tc_top -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_potrf_cm --launch-skip 100 -c 1 \
   -o gpurun_out/ncu_potrf_cm -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_simt --launch-skip 200 -c 1 \
   -o gpurun_out/ncu_gemm_simt -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/ncu3.log 2>&1
