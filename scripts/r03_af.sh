# full validation at HEAD: GPU tests, smoke, bench (both arms), launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_af.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_af.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke_af.log 2>&1; echo SMOKE $? >> gpurun_out/smoke_af.log
timeout 900 python bench.py > gpurun_out/bench_af.log 2> gpurun_out/bench_af.err; echo BENCH $? >> gpurun_out/bench_af.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_af.log 2> gpurun_out/bench_ref_af.err; echo REF $? >> gpurun_out/bench_ref_af.err
