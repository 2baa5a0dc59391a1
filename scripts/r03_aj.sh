# sharded Lloyd assignments (loopback ranks on one GPU) + the sharded solve tests
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_shard.py -q -x > gpurun_out/tests_aj.log 2>&1; echo TESTS $? >> gpurun_out/tests_aj.log
