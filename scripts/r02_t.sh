# r02: Nystrom factors built on the landmark job concurrently with the LSH k-means
mkdir -p gpurun_out
OMP_NUM_THREADS=$(nproc) timeout 1200 python -m pytest tests -q -x -m gpu -k "lcn or shard or nystrom or factor or staged or bp or runner" > gpurun_out/tests_t.log 2>&1; echo TESTS $? >> gpurun_out/tests_t.log
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/timing_t.log 2>&1; echo RC $? >> gpurun_out/timing_t.log
