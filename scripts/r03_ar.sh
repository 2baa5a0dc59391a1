# full validation at HEAD: GPU tests, smoke, bench (ours), TC launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_ar.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_ar.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke_ar.log 2>&1; echo SMOKE $? >> gpurun_out/smoke_ar.log
timeout 900 python bench.py > gpurun_out/bench_ar.log 2> gpurun_out/bench_ar.err; echo BENCH $? >> gpurun_out/bench_ar.err
