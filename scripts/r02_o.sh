# r02: sparse-only operator at configs[3] (timing), factorization-error test
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_staged.py -q -x -k factorization > gpurun_out/tests_o.log 2>&1; echo TESTS $? >> gpurun_out/tests_o.log
PROBE_SPARSE=1 timeout 300 python scripts/probe.py c3 1.0 2 > gpurun_out/probe_sparse_o.log 2>&1; echo RC $? >> gpurun_out/probe_sparse_o.log
