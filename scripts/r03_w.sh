# GEMM + top-2 filter for d > 128
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gemm or lloyd or assign or config1 or lcn_small" > gpurun_out/tests_w.log 2>&1; echo TESTS $? >> gpurun_out/tests_w.log
LCN_TIMING=1 timeout 300 python scripts/probe.py c1 1.0 1 > gpurun_out/timing_w.log 2>&1
LCN_FILTER=exact LCN_TIMING=1 timeout 300 python scripts/probe.py c1 1.0 1 > gpurun_out/timing_w0.log 2>&1
