# reduce kernel with exp once per partial: parity, timing, launch list; then full bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/t_r05d.log 2>&1; echo TESTS $? >> gpurun_out/t_r05d.log
timeout 600 python scripts/probe.py c3 1.0 4 2>&1 | grep -E "sinkhorn|phases" > gpurun_out/probe_r05d.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lowrank_reduce|iter_end" -s 100 -c 12 --csv --log-file gpurun_out/launches_reduce_r05d.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-c4 --no-dense --no-e2e --no-fp64 > gpurun_out/ncu_r05d.log 2>&1; echo NCU $? >> gpurun_out/ncu_r05d.log
timeout 900 python bench.py > gpurun_out/bench_r05d.log 2> gpurun_out/bench_r05d.err; echo BENCH $? >> gpurun_out/bench_r05d.err
