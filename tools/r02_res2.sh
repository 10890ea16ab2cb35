#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_res2.txt
: > $O
timeout 1200 python tools/opt_sweep.py --n 65536 --reps 3 --set "" --set crit_max_ctas=140 --set prio_levels=3,crit_max_ctas=140 --set prio_levels=3,crit_max_ctas=136 --set prio_levels=3,crit_max_ctas=128 --set prio_levels=3,crit_max_ctas=140,bulk_max_ctas=140,bulk_tiles_per_cta=0 >> $O 2>&1
timeout 300 python tools/trace_bins.py --n 65536 --opt prio_levels=3 --opt crit_max_ctas=140 --json gpurun_out/tr4_p3m140.json > /dev/null 2>&1
