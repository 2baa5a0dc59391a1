# PDL between the LCN iteration kernels: tests + A/B iteration rate
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_bp.py -q -x > gpurun_out/tests_ah.log 2>&1; echo TESTS $? >> gpurun_out/tests_ah.log
for v in 1 0 1 0; do
  LCN_ITER_PDL=$v timeout 300 python scripts/probe.py c3 1.0 3 2>&1 | grep -E "sinkhorn 100" | sed "s/^/PDL=$v /" >> gpurun_out/iter_ah.log
done
