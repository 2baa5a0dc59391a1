mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -k "lloyd or kmeans or lsh or shard or schedules or lcn_small" > gpurun_out/tests_an.log 2>&1; echo TESTS $? >> gpurun_out/tests_an.log
LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 3 > gpurun_out/e2e_an.log 2>&1
