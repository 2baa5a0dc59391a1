# Round-end check on one GPU: tests, smoke, both bench arms.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo SMOKE $? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2> gpurun_out/bench_final.err; echo BENCH $? >> gpurun_out/bench_final.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo REF $? >> gpurun_out/bench_ref.err
