# Later bands overlap the first band's tail (late programmatic wait): parity tests, A/B timing, iteration launch list.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_staged.py -m gpu -x -q > gpurun_out/t_r05c.log 2>&1; echo TESTS $? >> gpurun_out/t_r05c.log
for rep in 1 2; do
for ov in 0 1; do
  echo "== LCN_BAND_OVERLAP=$ov rep $rep" >> gpurun_out/ab_r05c.log
  LCN_BAND_OVERLAP=$ov timeout 600 python scripts/probe.py c3 1.0 4 2>&1 | grep -E "sinkhorn|phases" >> gpurun_out/ab_r05c.log
done; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"band_stream|lowrank|iter_end" -s 200 -c 60 --csv --log-file gpurun_out/launches_r05.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-c4 --no-dense --no-e2e --no-fp64 > gpurun_out/ncu_r05c.log 2>&1; echo NCU $? >> gpurun_out/ncu_r05c.log
