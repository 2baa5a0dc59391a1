# Lloyd with certified bounds: tests + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "kmeans_pp or lloyd or lsh_buckets or assign" > gpurun_out/tests_o.log 2>&1; echo TESTS $? >> gpurun_out/tests_o.log
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/timing_o.log 2>&1
timeout 300 python scripts/timeline.py 2000000 4096 2>&1 | grep -v Warn > gpurun_out/timeline_o.log
