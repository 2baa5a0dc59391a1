# batched seeding (LSH bands + landmarks in one step chain): full GPU suite + timing + bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_p.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_p.log
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/timing_p.log 2>&1
LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 3 > gpurun_out/e2e_p.log 2>&1
