#!/bin/bash
# scheduling knobs of the trailing updates vs graph time (development)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/sched.txt
for cfg in "bulk_tiles_per_cta=0" "bulk_tiles_per_cta=1" "bulk_tiles_per_cta=2" "bulk_max_ctas=132" "bulk_max_ctas=116" "n_streams=2" "n_streams=4" "n_streams=10" "use_graph=0"; do
  echo "$cfg" >> gpurun_out/sched.txt
  timeout 300 python tools/critpath.py --n 65536 --opt syrk_split_min=4096 --opt $cfg | head -1 | cut -c1-200 >> gpurun_out/sched.txt 2>&1
done
