# r02: int8 filter rows for the k-means++ seeding: bit-exact tests + C3 timing (int8 vs fp16)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -k "kmeans_pp or lsh or lloyd or assign or small_configs or sparse_config0" > gpurun_out/tests_n.log 2>&1; echo TESTS $? >> gpurun_out/tests_n.log
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/timing_n_i8.log 2>&1; echo RC $? >> gpurun_out/timing_n_i8.log
LCN_PP_FILTER=half LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/timing_n_half.log 2>&1; echo RC $? >> gpurun_out/timing_n_half.log
