#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/pair_test.py > gpurun_out/r02_pair.txt 2>&1; echo rc=$? >> gpurun_out/r02_pair.txt
nvidia-smi --query-gpu=index,clocks.sm,power.draw --format=csv >> gpurun_out/r02_pair.txt
