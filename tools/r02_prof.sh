#!/bin/bash
# round-2 measurement pass: bench lines (ours + reference arm), launch list of
# one bench step with DRAM bytes, full captures of the hot kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02p_bench.jsonl 2> gpurun_out/r02p_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02p_bench_reference.jsonl 2> gpurun_out/r02p_bench_reference.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02p_launches_bench.csv \
   python bench.py --steps 1 --warmup 0 --e2e-steps 0 --cpu-n 0 --c4-count 0 --no-variants > gpurun_out/r02p_bench_ncu.log 2>&1
TOP=$(python tools/critpath.py --n 65536 --ncu-pick)
MID=$(python tools/critpath.py --n 65536 --ncu-pick --pick-n 8192)
T32=$(python tools/critpath.py --n 65536 --ncu-pick --pick-class tc32)
echo "top $TOP mid $MID tc32 $T32" > gpurun_out/r02p_pick.txt
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
timeout 900 $NCU -k regex:k_gemm_tcILi0E --launch-skip $TOP -c 1 -o gpurun_out/r02p_gemm_tc_top -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/r02p_a.log 2>&1
timeout 900 $NCU -k regex:k_gemm_tcILi0E --launch-skip $MID -c 1 -o gpurun_out/r02p_gemm_tc_8192 -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/r02p_b.log 2>&1
timeout 900 $NCU -k regex:k_gemm_tcILi1E --launch-skip $T32 -c 1 -o gpurun_out/r02p_gemm_tc32 -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/r02p_c.log 2>&1
timeout 600 $NCU -k regex:k_potrf_v2 --launch-skip 20 -c 1 -o gpurun_out/r02p_potrf -f python tools/critpath.py --n 16384 --profile-only > gpurun_out/r02p_d.log 2>&1
timeout 600 $NCU -k regex:k_leaf_inv2 --launch-skip 20 -c 1 -o gpurun_out/r02p_inverse -f python tools/critpath.py --n 16384 --profile-only > gpurun_out/r02p_e.log 2>&1
timeout 600 $NCU -k regex:k_potrf_f64 --launch-skip 3 -c 1 -o gpurun_out/r02p_potrf_f64 -f python tools/critpath.py --n 8192 --cfg "[F16, F32, F64]" --profile-only > gpurun_out/r02p_f.log 2>&1
timeout 600 $NCU -k regex:k_export -c 1 --launch-skip 255 -o gpurun_out/r02p_export -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/r02p_g.log 2>&1
timeout 600 $NCU -k regex:k_quant1 -c 1 --launch-skip 0 -o gpurun_out/r02p_quant -f python tools/critpath.py --n 65536 --profile-only > gpurun_out/r02p_h.log 2>&1
timeout 600 $NCU -k regex:k_potrs_sweep -c 2 --launch-skip 2 -o gpurun_out/r02p_potrs -f python tools/potrs_bench.py > gpurun_out/r02p_i.log 2>&1
timeout 300 python tools/potrs_bench.py > gpurun_out/r02p_potrs_bench.txt 2>&1
timeout 300 python tools/fp64_peak.py gpurun_out/r02p_fp64_peak.json > /dev/null 2>&1
