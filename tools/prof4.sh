#!/bin/bash
# profiling pass (round 1, final): launch list of the bench command with DRAM
# bytes, full captures of the hot kernels of every class
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bench3.csv \
   python bench.py --steps 1 --warmup 0 --e2e-steps 0 --cpu-n 0 --c4-count 0 > gpurun_out/bench_ncu3.log 2>&1
IDX=$(python tools/critpath.py --n 65536 --ncu-pick)
echo "pick $IDX" > gpurun_out/ncu4_pick.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc --launch-skip $IDX -c 1 \
   -o gpurun_out/ncu4_gemm_tc_top -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/ncu4a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:k_potrf_v2 --launch-skip 20 -c 1 \
   -o gpurun_out/ncu4_potrf -f python tools/critpath.py --n 16384 --profile-only > gpurun_out/ncu4b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_quant1 -c 1 --launch-skip 7 \
   -o gpurun_out/ncu4_quant -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/ncu4c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_potrs_sweep -c 1 --launch-skip 2 \
   -o gpurun_out/ncu4_potrs -f python tools/potrs_bench.py > gpurun_out/ncu4d.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leaf_inv2 --launch-skip 20 -c 1 \
   -o gpurun_out/ncu4_inverse -f python tools/critpath.py --n 16384 --profile-only > gpurun_out/ncu4e.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_import -c 1 --launch-skip 375 \
   -o gpurun_out/ncu4_import -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/ncu4f.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_export -c 1 --launch-skip 255 \
   -o gpurun_out/ncu4_export -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/ncu4g.log 2>&1
