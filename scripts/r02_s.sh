# r02: k-means++ filter with register-loaded rows: bit-exact tests + C3 seeding timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -k "kmeans_pp or lsh_buckets or lloyd or small_configs" > gpurun_out/tests_s.log 2>&1; echo TESTS $? >> gpurun_out/tests_s.log
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/timing_s.log 2>&1; echo RC $? >> gpurun_out/timing_s.log
