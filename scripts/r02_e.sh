# r02: full configs[1], configs[3]@0.1 and 5000^2 dense parity vs the compiled reference
mkdir -p gpurun_out
nproc > gpurun_out/host_e.txt
OMP_NUM_THREADS=$(nproc) timeout 2400 python -m pytest tests/test_gpu_parity.py -q -x -k "large_configs or dense_anchor" --durations=10 > gpurun_out/large_tests.log 2>&1; echo TESTS $? >> gpurun_out/large_tests.log
