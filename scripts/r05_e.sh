# e2e leg: phase timings, band overlap on/off, then the bench's e2e leg twice
mkdir -p gpurun_out
nproc > gpurun_out/e2e_r05e.log; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/e2e_r05e.log; free -g | head -2 >> gpurun_out/e2e_r05e.log
for ov in 1 0; do
  echo "== LCN_BAND_OVERLAP=$ov" >> gpurun_out/e2e_r05e.log
  LCN_BAND_OVERLAP=$ov LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 4 >> gpurun_out/e2e_r05e.log 2>&1
done
for k in 1 2; do
timeout 900 python bench.py --no-cpu --no-c4 --no-dense --no-fp64 > gpurun_out/bench_r05e_$k.log 2> gpurun_out/bench_r05e_$k.err; echo BENCH $? >> gpurun_out/bench_r05e_$k.err
done
