mkdir -p gpurun_out
LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 4 > gpurun_out/e2e_s.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_s.log 2> gpurun_out/bench_s.err; echo BENCH $? >> gpurun_out/bench_s.err
