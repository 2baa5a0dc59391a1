mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_staged.py tests/test_gpu_integration.py tests/test_gpu_runner.py -q -x > gpurun_out/tests_al.log 2>&1; echo TESTS $? >> gpurun_out/tests_al.log
LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 3 > gpurun_out/e2e_al.log 2>&1
