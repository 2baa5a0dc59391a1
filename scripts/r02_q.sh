# r02: U / V from fp64 cuBLAS GEMMs in the fp32-storage build: parity + timing, sparse bench entry smoke
mkdir -p gpurun_out
OMP_NUM_THREADS=$(nproc) timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -k "lcn or shard or nystrom or multihead or grad or plan" > gpurun_out/tests_q.log 2>&1; echo TESTS $? >> gpurun_out/tests_q.log
timeout 300 python tests/parity_c3_gpu.py gpurun_out/parity_s005_q.npz 0.005 > gpurun_out/parity_s005_q.log 2>&1; echo RC $? >> gpurun_out/parity_s005_q.log
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/timing_q.log 2>&1; echo RC $? >> gpurun_out/timing_q.log
