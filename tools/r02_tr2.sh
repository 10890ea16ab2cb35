#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/trace_bins.py --n 65536 --json gpurun_out/tr_default.json > /dev/null 2>&1
timeout 300 python tools/trace_bins.py --n 65536 --opt trsm_row_split_min=4096 --opt syrk_split_min=4096 --json gpurun_out/tr_split.json > /dev/null 2>&1
timeout 300 python tools/trace_bins.py --n 16384 --json gpurun_out/tr_16384.json > /dev/null 2>&1
