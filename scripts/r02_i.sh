# r02: full configs[2] parity, bench (ours), reference arm
mkdir -p gpurun_out
OMP_NUM_THREADS=$(nproc) timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config2_full" --durations=3 > gpurun_out/c2full.log 2>&1; echo TESTS $? >> gpurun_out/c2full.log
timeout 1200 python bench.py > gpurun_out/bench_i.log 2>&1; echo RC $? >> gpurun_out/bench_i.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref_i.log 2>&1; echo RC $? >> gpurun_out/bench_ref_i.log
