# r02: refresh: full GPU suite, bench (ours + reference arm), launch list + band traffic capture
mkdir -p gpurun_out
OMP_NUM_THREADS=$(nproc) timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_u.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_u.log
timeout 1200 python bench.py > gpurun_out/bench_u.log 2>&1; echo RC $? >> gpurun_out/bench_u.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref_u.log 2>&1; echo RC $? >> gpurun_out/bench_ref_u.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"band_stream|lowrank|iter_end|shard_" -s 40 -c 24 --csv --log-file gpurun_out/launches_u.csv python scripts/probe.py c3 1.0 1 > gpurun_out/launches_u.log 2>&1; echo RC $? >> gpurun_out/launches_u.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_stream_kernel -s 8 -c 4 -o gpurun_out/prof_band_u -f python scripts/probe.py c3 1.0 1 > gpurun_out/prof_band_u.log 2>&1; echo RC $? >> gpurun_out/prof_band_u.log
