# single-CTA certified pick + PDL chain: tests, timeline, build timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "kmeans_pp or lloyd or lsh_buckets" > gpurun_out/tests_e.log 2>&1; echo TESTS $? >> gpurun_out/tests_e.log
LCN_PP_PDL=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "kmeans_pp" >> gpurun_out/tests_e.log 2>&1; echo TESTS_NOPDL $? >> gpurun_out/tests_e.log
for v in "LCN_PP_PDL=1" "LCN_PP_PDL=0"; do
  echo "== $v" >> gpurun_out/timeline_e.log
  env $v timeout 300 python scripts/timeline.py 2000000 4096 2>&1 | grep -v Warn >> gpurun_out/timeline_e.log
done
for v in "LCN_PP_FILTER=f16" "LCN_PP_FILTER=i8"; do
  echo "== $v" >> gpurun_out/timing_e.log
  env $v LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 2>&1 | grep -E "timed|seeding|lsh k-means|^build|fallback" >> gpurun_out/timing_e.log
done
