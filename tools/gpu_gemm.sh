#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/gemm_bench.py tc16 tc32 simt_f32 > gpurun_out/gemm_bench.txt 2>&1
timeout 300 ncu --set full --import-source on -k regex:k_gemm_tc --launch-skip 1 -c 1 -o gpurun_out/ncu_gemm_small -f \
  python -c "import sys; sys.path.insert(0,'.'); import paper_2601_08082_b200 as tc; tc.debug_gemm('tc16', 8192, 256, 512, False, 0.0, 0, 1)" > gpurun_out/ncu_small.log 2>&1
timeout 300 ncu --set full --import-source on -k regex:k_trsm_cm --launch-skip 3 -c 1 -o gpurun_out/ncu_trsm_cm -f \
  python tools/critpath.py --n 16384 --profile-only > gpurun_out/ncu_trsm.log 2>&1
