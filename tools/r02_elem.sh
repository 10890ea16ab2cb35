#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_elem.txt
: > $O
timeout 1500 python tools/opt_sweep.py --n 65536 --reps 3 --set g:elem_tiles_per_cta=0 --set g:elem_tiles_per_cta=4,node_prio=1,import_low=1 --set g:elem_tiles_per_cta=4,node_prio=1,import_low=1,prio_levels=3 --set g:elem_tiles_per_cta=1,node_prio=1,import_low=1,prio_levels=3 --set g:elem_tiles_per_cta=4,node_prio=1,import_low=1,prio_levels=3,crit_max_ctas=140 --set g:elem_tiles_per_cta=4 >> $O 2>&1
timeout 300 python tools/trace_bins.py --n 65536 --opt g:elem_tiles_per_cta=4 --opt node_prio=1 --opt import_low=1 --opt prio_levels=3 --json gpurun_out/tr7.json > /dev/null 2>&1
