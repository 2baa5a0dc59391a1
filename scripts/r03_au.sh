# Lloyd tile skipping
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "lloyd or assign or lsh_buckets" > gpurun_out/tests_au.log 2>&1; echo TESTS $? >> gpurun_out/tests_au.log
LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 3 > gpurun_out/e2e_au.log 2>&1
