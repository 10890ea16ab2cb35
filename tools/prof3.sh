#!/bin/bash
# targeted captures: the top FP16 GEMM (by flops), the largest quantize /
# import / export launches (HBM-bound kernels), the F64 DMMA GEMM
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
IDX=$(python tools/critpath.py --n 65536 --ncu-pick)
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_gemm_tc<0>" --launch-skip $IDX -c 1 \
   -o gpurun_out/ncu3_gemm_tc_top -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/ncu3a.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_quant1 --launch-skip 2 -c 1 \
   -o gpurun_out/ncu3_quant_top -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/ncu3b.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_export --launch-skip 255 -c 1 \
   -o gpurun_out/ncu3_export_big -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/ncu3c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_dmma -c 1 --launch-skip 3 \
   -o gpurun_out/ncu3_dmma -f python tools/critpath.py --n 8192 --cfg "Pure F64" --profile-only > gpurun_out/ncu3d.log 2>&1
timeout 600 python tools/gemm_bench.py simt_f64 > gpurun_out/gemm_f64.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
