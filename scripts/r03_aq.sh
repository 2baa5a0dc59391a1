mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:assign_filter_tc -c 2 --csv python scripts/tc_bench.py 2000000 4096 0 > gpurun_out/tc_aq.csv 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -k "assign or lloyd or lsh or kmeans or shard or schedules or lcn_small" > gpurun_out/tests_aq.log 2>&1; echo TESTS $? >> gpurun_out/tests_aq.log
LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 3 > gpurun_out/e2e_aq.log 2>&1
