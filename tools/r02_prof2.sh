#!/bin/bash
# round-2 final measurement pass (after CTA pairs and fused leaf shadows)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02q_bench.jsonl 2> gpurun_out/r02q_bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02q_launches_bench.csv \
   python bench.py --steps 1 --warmup 0 --e2e-steps 0 --cpu-n 0 --c4-count 0 --no-variants > gpurun_out/r02q_bench_ncu.log 2>&1
TOP=$(python tools/critpath.py --n 65536 --ncu-pick)
echo "top $TOP" > gpurun_out/r02q_pick.txt
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:k_gemm_tc2 -c 1 -o gpurun_out/r02q_gemm_tc2_first -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/r02q_a.log 2>&1
timeout 900 $NCU -k regex:k_gemm_tc2 --launch-skip 40 -c 1 -o gpurun_out/r02q_gemm_tc2_mid -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/r02q_b.log 2>&1
timeout 600 python tools/critpath.py --n 65536 --json gpurun_out/r02q_crit65536.json > gpurun_out/r02q_crit65536.txt 2>&1
timeout 300 python tools/critpath.py --n 16384 > gpurun_out/r02q_crit16384.txt 2>&1
timeout 600 python tools/gemm_ops.py 65536 > gpurun_out/r02q_gemm_ops_65536.txt 2>&1
