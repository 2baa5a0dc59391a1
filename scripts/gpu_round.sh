# Round-end style GPU pass: tests, bench, ncu launch list + full capture of the band kernel.
# usage (on the GPU box): bash scripts/gpu_round.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2> gpurun_out/bench_$TAG.err; echo BENCH $? >> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"band_stream|lowrank|iter_end" -c 16 --csv --log-file gpurun_out/launches_$TAG.csv \
  python scripts/probe.py c3 1.0 1 > gpurun_out/ncu_list_$TAG.log 2>&1; echo NCU1 $? >> gpurun_out/ncu_list_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_stream -c 4 \
  -o gpurun_out/prof_band_full_$TAG -f python scripts/probe.py c3 1.0 1 > gpurun_out/ncu_full_$TAG.log 2>&1; echo NCU2 $? >> gpurun_out/ncu_full_$TAG.log
