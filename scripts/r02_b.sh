# r02: bucket-sharded solve (loopback ranks on one GPU) + the full GPU suite
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_parity.py -k "shard" -q > gpurun_out/gpu_shard.log 2>&1; echo TESTS $? >> gpurun_out/gpu_shard.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_b.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_b.log
