# landmarks seeded in the bands' batch, the early job waits on that sequence's event
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_staged.py tests/test_gpu_runner.py tests/test_gpu_lsh_schemes.py -q -x > gpurun_out/tests_as.log 2>&1; echo TESTS $? >> gpurun_out/tests_as.log
LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 3 > gpurun_out/e2e_as.log 2>&1
