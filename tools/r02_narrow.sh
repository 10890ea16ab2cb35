#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/narrow_test.py > gpurun_out/r02_narrow.txt 2>&1
echo rc=$? >> gpurun_out/r02_narrow.txt
timeout 1200 python tools/opt_sweep.py --n 65536 --reps 3 --set "" --set g:tc_narrow_max_tiles=148 --set g:tc_narrow_max_tiles=296 >> gpurun_out/r02_narrow.txt 2>&1
timeout 400 python tools/opt_sweep.py --n 16384 --reps 3 --set "" --set g:tc_narrow_max_tiles=148 --set g:tc_narrow_max_tiles=296 >> gpurun_out/r02_narrow.txt 2>&1
