# round-end style pass: all GPU tests, smoke, bench (ours), launch list, band capture
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_ab.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_ab.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke_ab.log 2>&1; echo SMOKE $? >> gpurun_out/smoke_ab.log
timeout 900 python bench.py > gpurun_out/bench_ab.log 2> gpurun_out/bench_ab.err; echo BENCH $? >> gpurun_out/bench_ab.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"band_stream|lowrank|iter_end" -c 16 --csv --log-file gpurun_out/launches_ab.csv \
  python scripts/probe.py c3 1.0 1 > gpurun_out/ncu_list_ab.log 2>&1; echo NCU1 $? >> gpurun_out/ncu_list_ab.log
