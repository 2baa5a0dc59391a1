# K_sp + CSR during the host LDL^T; parallel LDL^T steps
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_t.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_t.log
LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 3 > gpurun_out/e2e_t.log 2>&1
