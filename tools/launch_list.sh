cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --replay-mode application --clock-control none --csv --log-file gpurun_out/launches_bench3.csv \
   python bench.py --steps 1 --warmup 0 --e2e-steps 0 --cpu-n 0 --c4-count 0 > gpurun_out/bench_ncu3.log 2>&1
echo rc=$? >> gpurun_out/bench_ncu3.log
