#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_imp.txt
: > $O
timeout 1500 python tools/opt_sweep.py --n 65536 --reps 3 --set "" --set node_prio=1,import_low=1 --set node_prio=1,prio_levels=3,import_low=1 --set node_prio=1,prio_levels=3,import_low=1,crit_max_ctas=140 --set node_prio=1,prio_levels=3,import_low=1,crit_max_ctas=140,trsm_row_split_min=4096,syrk_split_min=4096 >> $O 2>&1
timeout 400 python tools/opt_sweep.py --n 16384 --reps 3 --set "" --set node_prio=1,import_low=1 --set node_prio=1,prio_levels=3,import_low=1 >> $O 2>&1
timeout 300 python tools/trace_bins.py --n 65536 --opt node_prio=1 --opt prio_levels=3 --opt import_low=1 --opt crit_max_ctas=140 --json gpurun_out/tr6.json > gpurun_out/tr6_bins.txt 2>&1
