# full GPU suite + bench after the seeding work
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_l.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_l.log
timeout 900 python bench.py > gpurun_out/bench_l.log 2> gpurun_out/bench_l.err; echo BENCH $? >> gpurun_out/bench_l.err
