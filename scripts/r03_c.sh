# split filter (filter -> survivors -> exact) vs fused; fp16 vs int8 rows
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "kmeans_pp or lloyd or lsh_buckets" > gpurun_out/tests_c.log 2>&1; echo TESTS $? >> gpurun_out/tests_c.log
LCN_PP_FILTER=i8 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "kmeans_pp" >> gpurun_out/tests_c.log 2>&1; echo TESTS_I8 $? >> gpurun_out/tests_c.log
for v in "LCN_PP_SPLIT=0" "LCN_PP_SPLIT=1" "LCN_PP_FILTER=i8"; do
  echo "== $v" >> gpurun_out/timing_c.log
  env $v LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 2>&1 | grep -E "timed|seeding|lsh k-means|^build" >> gpurun_out/timing_c.log
done
