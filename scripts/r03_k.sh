# persistent prune + int8 filter scan
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "kmeans_pp or lloyd or lsh_buckets" > gpurun_out/tests_k.log 2>&1; echo TESTS $? >> gpurun_out/tests_k.log
LCN_PP_SCAN=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "kmeans_pp" >> gpurun_out/tests_k.log 2>&1; echo TESTS_NOSCAN $? >> gpurun_out/tests_k.log
LCN_PP_PDL=0 timeout 300 python scripts/timeline.py 2000000 4096 2>&1 | grep -v Warn > gpurun_out/timeline_k0.log
timeout 300 python scripts/timeline.py 2000000 4096 2>&1 | grep -v Warn > gpurun_out/timeline_k.log
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/timing_k.log 2>&1
