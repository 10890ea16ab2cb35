#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02_pytest_full.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo rc=$? >> gpurun_out/r02_smoke.log
timeout 900 python bench.py > gpurun_out/r02_bench3.jsonl 2> gpurun_out/r02_bench3.err
