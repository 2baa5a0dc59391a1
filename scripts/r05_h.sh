# Final check at HEAD on one GPU: tests, smoke, both bench arms.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_r05h.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_r05h.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke_r05h.log 2>&1; echo SMOKE $? >> gpurun_out/smoke_r05h.log
timeout 900 python bench.py > gpurun_out/bench_r05h.log 2> gpurun_out/bench_r05h.err; echo BENCH $? >> gpurun_out/bench_r05h.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r05h.log 2> gpurun_out/bench_ref_r05h.err; echo REF $? >> gpurun_out/bench_ref_r05h.err
for rep in 1 2 3 4 5 6; do
  s0=$SECONDS
  timeout -s ABRT 150 python -X faulthandler bench.py --no-e2e --no-cpu --no-c4 --no-dense --no-fp64 > gpurun_out/stallh_${rep}.log 2> gpurun_out/stallh_${rep}.err
  echo "default rep=$rep rc=$? wall=$((SECONDS - s0))" >> gpurun_out/stall_r05h.log
done
