#!/bin/bash
# profiling pass (round 1, after tuning): launch list of the bench command,
# full captures of the top kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bench2.csv \
   python bench.py --steps 1 --warmup 0 --e2e-steps 0 --cpu-n 0 --c4-count 0 > gpurun_out/bench_ncu2.log 2>&1
IDX=$(python tools/critpath.py --n 65536 --ncu-pick)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc --launch-skip $IDX -c 1 \
   -o gpurun_out/ncu2_gemm_tc_top -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/ncu2a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_potrf_v2 --launch-skip 20 -c 1 \
   -o gpurun_out/ncu2_potrf -f python tools/critpath.py --n 16384 --profile-only > gpurun_out/ncu2b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc --launch-skip 40 -c 1 \
   -o gpurun_out/ncu2_gemm_small -f python tools/critpath.py --n 16384 --profile-only > gpurun_out/ncu2c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_quant1 -c 1 \
   -o gpurun_out/ncu2_quant -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/ncu2d.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_potrs_fwd -c 1 \
   -o gpurun_out/ncu2_potrs -f python tools/potrs_bench.py > gpurun_out/ncu2e.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leaf_inv2 --launch-skip 20 -c 1 \
   -o gpurun_out/ncu2_inverse -f python tools/critpath.py --n 16384 --profile-only > gpurun_out/ncu2f.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_import -c 1 --launch-skip 100 \
   -o gpurun_out/ncu2_import -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/ncu2g.log 2>&1
