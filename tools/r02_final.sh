#!/bin/bash
# round-2 final measurement pass: GPU tests, smoke, bench lines (ours +
# reference arm), launch list of one bench step with DRAM bytes, full
# captures of the CTA-pair GEMMs (both kinds) and a single-CTA FP16 launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=gpurun_out/r02z
timeout 1500 python -m pytest tests -q -m gpu > ${P}_pytest.log 2>&1; echo rc=$? >> ${P}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${P}_smoke.txt 2>&1
timeout 900 python bench.py > ${P}_bench.jsonl 2> ${P}_bench.err
timeout 600 python bench.py --impl reference > ${P}_bench_reference.jsonl 2> ${P}_bench_reference.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file ${P}_launches_bench.csv \
   python bench.py --steps 1 --warmup 0 --e2e-steps 0 --cpu-n 0 --c4-count 0 --no-variants > ${P}_bench_ncu.log 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
timeout 900 $NCU -k regex:k_gemm_tc2ILi0E -c 1 -o ${P}_gemm_tc2_first -f python tools/critpath.py --n 65536 --profile-only > ${P}_a.log 2>&1
timeout 900 $NCU -k regex:k_gemm_tc2ILi0E --launch-skip 40 -c 1 -o ${P}_gemm_tc2_mid -f python tools/critpath.py --n 65536 --profile-only > ${P}_b.log 2>&1
timeout 900 $NCU -k regex:k_gemm_tc2ILi1E -c 1 -o ${P}_gemm_tc2_tf32 -f python tools/critpath.py --n 65536 --profile-only > ${P}_c.log 2>&1
timeout 900 $NCU -k regex:k_gemm_tcILi0E --launch-skip 200 -c 1 -o ${P}_gemm_tc_mid -f python tools/critpath.py --n 65536 --profile-only > ${P}_d.log 2>&1
timeout 600 $NCU -k regex:k_potrf_v2 --launch-skip 20 -c 1 -o ${P}_potrf -f python tools/critpath.py --n 16384 --profile-only > ${P}_e.log 2>&1
