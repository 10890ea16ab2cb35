#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02r_bench.jsonl 2> gpurun_out/r02r_bench.err
timeout 300 python tools/gemm_ops.py 16384 > gpurun_out/r02r_gemm_ops_16384.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02r_smoke.txt 2>&1
