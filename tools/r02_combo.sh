#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_combo.txt
: > $O
S="trsm_row_split_min=4096,syrk_split_min=4096"
R="node_prio=1,prio_levels=3,crit_max_ctas=136,bulk_max_ctas=136"
timeout 1500 python tools/opt_sweep.py --n 65536 --reps 3 --set "" --set $R,bulk_tiles_per_cta=0 --set $R,bulk_tiles_per_cta=0,$S --set $R,bulk_tiles_per_cta=4,$S --set node_prio=1,prio_levels=3,crit_max_ctas=128,bulk_max_ctas=128,bulk_tiles_per_cta=0,$S >> $O 2>&1
