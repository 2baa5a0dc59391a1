# landmarks + Nystrom factors on an early job beside the bands' seeding chain
mkdir -p gpurun_out
for v in "LCN_EARLY_FACTORS=1" "LCN_EARLY_FACTORS=0"; do
  echo "== $v" >> gpurun_out/e2e_ae.log
  env $v LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 3 >> gpurun_out/e2e_ae.log 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_staged.py tests/test_gpu_bp.py tests/test_gpu_integration.py -q -x > gpurun_out/tests_ae.log 2>&1; echo TESTS $? >> gpurun_out/tests_ae.log
