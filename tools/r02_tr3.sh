#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/trace_bins.py --n 65536 --json gpurun_out/tr3_default.json > /dev/null 2>&1
timeout 300 python tools/trace_bins.py --n 65536 --opt prio_levels=3 --json gpurun_out/tr3_prio3.json > /dev/null 2>&1
timeout 300 python tools/trace_bins.py --n 65536 --opt prio_levels=3 --opt crit_max_ctas=140 --json gpurun_out/tr3_prio3m140.json > /dev/null 2>&1
