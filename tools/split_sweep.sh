cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for v in 0 8192 4096 2048 1024; do
  echo "split=$v" >> gpurun_out/split.txt
  timeout 300 python tools/critpath.py --n 65536 --opt syrk_split_min=$v | head -1 >> gpurun_out/split.txt 2>&1
  timeout 300 python tools/critpath.py --n 16384 --opt syrk_split_min=$v | head -1 >> gpurun_out/split.txt 2>&1
done
