#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_prio.txt
: > $O
timeout 900 python tools/opt_sweep.py --n 65536 --reps 3 --set "" --set prio_levels=3 --set prio_levels=3,crit_tiles_per_cta=1 --set prio_levels=3,crit_tiles_per_cta=4 --set prio_levels=3,crit_max_ctas=144 --set prio_levels=3,trsm_row_split_min=4096,syrk_split_min=4096 --set prio_levels=3,crit_tiles_per_cta=2,trsm_row_split_min=4096,syrk_split_min=4096 >> $O 2>&1
timeout 300 python tools/opt_sweep.py --n 16384 --reps 3 --set "" --set prio_levels=3 --set prio_levels=3,crit_tiles_per_cta=1 >> $O 2>&1
timeout 300 python tools/trace_bins.py --n 65536 --opt prio_levels=3 --json gpurun_out/tr_prio3.json > /dev/null 2>&1
timeout 300 python tools/trace_bins.py --n 65536 --opt prio_levels=3 --opt crit_tiles_per_cta=1 --json gpurun_out/tr_prio3c1.json > /dev/null 2>&1
