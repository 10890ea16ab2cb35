#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_tiles.txt
timeout 300 python tools/potrf_clk.py > $O 2>&1
timeout 300 python tools/leafclk.py >> $O 2>&1
timeout 900 python tools/opt_sweep.py --n 65536 --reps 4 --set "" --set bulk_tiles_per_cta=2 --set bulk_tiles_per_cta=4 --set bulk_tiles_per_cta=0 >> $O 2>&1
timeout 600 python tools/opt_sweep.py --n 16384 --reps 7 --set "" --set bulk_tiles_per_cta=2 --set bulk_tiles_per_cta=0 >> $O 2>&1
timeout 600 python tools/c4_bench.py 16,32 16,32,bulk_tiles_per_cta=2 16,32,bulk_tiles_per_cta=4 >> $O 2>&1
timeout 600 python -m pytest tests -x -q -m gpu -k "factor or inverse" > gpurun_out/r02_pytest_inv.log 2>&1; echo rc=$? >> gpurun_out/r02_pytest_inv.log
