# prune 512x4 (32 regs), squared test; exact grid 1/SM/sequence
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_runner.py tests/test_gpu_lsh_schemes.py -q -x -k "kmeans_pp or lloyd or lsh or runner" > gpurun_out/tests_q.log 2>&1; echo TESTS $? >> gpurun_out/tests_q.log
LCN_PP_PDL=0 timeout 300 python scripts/timeline.py 2000000 4096 2>&1 | grep -v Warn > gpurun_out/timeline_q0.log
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/timing_q.log 2>&1
