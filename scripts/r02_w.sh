# r02: bench through the NCCL bucket-sharded path at N = 1 (--sharded), reduced extras
mkdir -p gpurun_out
timeout 900 python bench.py --sharded --steps 5 --warmup 3 --no-c4 --no-dense --no-cpu --no-fp64 > gpurun_out/bench_sharded_w.log 2>&1; echo RC $? >> gpurun_out/bench_sharded_w.log
