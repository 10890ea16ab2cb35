#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_narrow3.txt
: > $O
timeout 1200 python tools/opt_sweep.py --n 65536 --reps 4 --set g:tc_narrow_max_tiles=0 --set g:tc_narrow_max_tiles=65 --set g:tc_narrow_max_tiles=0 --set g:tc_narrow_max_tiles=65 >> $O 2>&1
timeout 400 python tools/opt_sweep.py --n 16384 --reps 4 --set g:tc_narrow_max_tiles=0 --set g:tc_narrow_max_tiles=65 --set g:tc_narrow_max_tiles=100 >> $O 2>&1
for v in 0 65 0 65; do echo -n "narrow=$v " >> $O; timeout 300 python tools/c4_bench.py 16,32,g:tc_narrow_max_tiles=$v >> $O 2>&1; done
