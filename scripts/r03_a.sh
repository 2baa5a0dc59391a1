# re-entry check at HEAD: GPU tests, smoke, bench (our arm)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_a.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_a.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke_a.log 2>&1; echo SMOKE $? >> gpurun_out/smoke_a.log
timeout 900 python bench.py > gpurun_out/bench_a.log 2> gpurun_out/bench_a.err; echo BENCH $? >> gpurun_out/bench_a.err
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/timing_a.log 2>&1; echo RC $? >> gpurun_out/timing_a.log
