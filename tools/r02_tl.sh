#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/timeline_bins.py --n 65536 --bin 4 > gpurun_out/r02_tlbins65536.txt 2>&1
timeout 300 python tools/timeline_bins.py --n 16384 --bin 0.5 > gpurun_out/r02_tlbins16384.txt 2>&1
timeout 300 python tools/timeline.py --n 65536 > gpurun_out/r02_tl65536.txt 2>&1
