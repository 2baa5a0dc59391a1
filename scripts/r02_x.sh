# r02: sharded finish on the device + lazy global support: shard tests + sharded bench at N = 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_parity.py -q -x -k "shard" > gpurun_out/tests_x.log 2>&1; echo TESTS $? >> gpurun_out/tests_x.log
timeout 900 python bench.py --sharded --steps 5 --warmup 3 --no-c4 --no-dense --no-cpu --no-fp64 > gpurun_out/bench_sharded_x.log 2>&1; echo RC $? >> gpurun_out/bench_sharded_x.log
