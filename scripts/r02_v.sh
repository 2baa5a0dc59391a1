# r02: dense recompute with N = 256 items: parity + timing
mkdir -p gpurun_out
OMP_NUM_THREADS=$(nproc) timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dense_recompute or dense_config2" > gpurun_out/tests_v.log 2>&1; echo TESTS $? >> gpurun_out/tests_v.log
LCN_DENSE_RECOMPUTE=1 timeout 300 python scripts/probe_dense.py 1.0 > gpurun_out/probe_dense_v.log 2>&1; echo RC $? >> gpurun_out/probe_dense_v.log
