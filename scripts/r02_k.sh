# r02: full GPU suite, bench (ours + reference arm), ncu of the dense recompute kernel
mkdir -p gpurun_out
OMP_NUM_THREADS=$(nproc) timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_k.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_k.log
timeout 1200 python bench.py > gpurun_out/bench_k.log 2>&1; echo RC $? >> gpurun_out/bench_k.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref_k.log 2>&1; echo RC $? >> gpurun_out/bench_ref_k.log
LCN_DENSE_RECOMPUTE=1 PROBE_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_lse_tc -c 1 -o gpurun_out/prof_dense_tc -f python scripts/probe_dense.py 1.0 > gpurun_out/prof_dense_tc.log 2>&1; echo RC $? >> gpurun_out/prof_dense_tc.log
