#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_nolook.txt
timeout 300 python tools/potrf_clk.py > $O 2>&1
(cd variants/nolook && timeout 300 python ../../tools/potrf_clk.py >> ../../$O 2>&1)
timeout 300 python tools/opt_sweep.py --n 16384 --reps 7 --set "" >> $O 2>&1
TC_ROOT=$GRAFT_REPO_ROOT/variants/nolook timeout 300 python tools/opt_sweep.py --n 16384 --reps 7 --set "" >> $O 2>&1
