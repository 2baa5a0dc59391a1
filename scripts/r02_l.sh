# r02: dense recompute v2 (TMEM-direct epilogue, 3 stages) + cuBLAS W GEMM: tests and timings
mkdir -p gpurun_out
OMP_NUM_THREADS=$(nproc) timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_staged.py -q -x -k "dense or lcn_large or staged or small_configs or wide or factor or nystrom" > gpurun_out/tests_l.log 2>&1; echo TESTS $? >> gpurun_out/tests_l.log
LCN_DENSE_RECOMPUTE=1 timeout 300 python scripts/probe_dense.py 1.0 > gpurun_out/probe_dense_l.log 2>&1; echo RC $? >> gpurun_out/probe_dense_l.log
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/timing_l.log 2>&1; echo RC $? >> gpurun_out/timing_l.log
