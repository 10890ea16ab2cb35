#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_pair2.txt
timeout 1500 python tools/opt_sweep.py --n 65536 --reps 4 --set "" --set g:tc_pair_min_tiles=128 --set g:tc_pair_min_tiles=256 --set g:tc_pair_min_tiles=512 --set g:tc_pair_min_tiles=2048 > $O 2>&1
timeout 600 python tools/opt_sweep.py --n 16384 --reps 7 --set "" --set g:tc_pair_min_tiles=128 --set g:tc_pair_min_tiles=256 --set g:tc_pair_min_tiles=512 >> $O 2>&1
timeout 900 python tools/c4_bench.py 16,32 16,32,g:tc_pair_min_tiles=256 16,32,g:tc_pair_min_tiles=512 >> $O 2>&1
