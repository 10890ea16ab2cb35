cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | grep -v "^  " | head -60
CUDA_LAUNCH_BLOCKING=1 timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/one.py 2>&1 | head -60
