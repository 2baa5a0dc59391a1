# HEAD check: GPU tests, smoke, bench line (ours).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r04a.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_r04a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r04a.log 2>&1; echo SMOKE $? >> gpurun_out/smoke_r04a.log
timeout 900 python bench.py > gpurun_out/bench_r04a.log 2> gpurun_out/bench_r04a.err; echo BENCH $? >> gpurun_out/bench_r04a.err
