#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r02_c4rep.txt
: > $O
timeout 600 python tools/c4_repeat.py 16 32 8 >> $O 2>&1
timeout 600 python tools/c4_repeat.py 32 32 6 >> $O 2>&1
timeout 600 python tools/c4_repeat.py 24 48 5 >> $O 2>&1
