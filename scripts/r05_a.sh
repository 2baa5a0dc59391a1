# Round-2 re-entry check at HEAD on one GPU: tests, smoke, both bench arms, ncu launch list.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_r05a.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_r05a.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke_r05a.log 2>&1; echo SMOKE $? >> gpurun_out/smoke_r05a.log
timeout 900 python bench.py > gpurun_out/bench_r05a.log 2> gpurun_out/bench_r05a.err; echo BENCH $? >> gpurun_out/bench_r05a.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r05a.log 2> gpurun_out/bench_ref_r05a.err; echo REF $? >> gpurun_out/bench_ref_r05a.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r05a.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_r05a.log 2>&1; echo NCU $? >> gpurun_out/ncu_r05a.log
