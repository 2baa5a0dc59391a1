# tc work counter test + e2e phase breakdown at HEAD + bench (distance roofline from the counter)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tc_work or tile_skipping or lloyd" > gpurun_out/t_r04b.log 2>&1; echo TESTS $? >> gpurun_out/t_r04b.log
LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 3 > gpurun_out/e2e_r04b.log 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/bench_r04b.log 2> gpurun_out/bench_r04b.err; echo BENCH $? >> gpurun_out/bench_r04b.err
