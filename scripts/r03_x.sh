mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gemm or lloyd" > gpurun_out/tests_x.log 2>&1; echo TESTS $? >> gpurun_out/tests_x.log
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c1 1.0 1 > gpurun_out/timing_x.log 2>&1
LCN_FILTER=exact LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c1 1.0 1 > gpurun_out/timing_x0.log 2>&1
