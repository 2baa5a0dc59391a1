mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -k "assign or lloyd or lsh or kmeans or shard or lcn_small" > gpurun_out/tests_at.log 2>&1; echo TESTS $? >> gpurun_out/tests_at.log
timeout 300 python scripts/timeline.py 2000000 4096 2>&1 | grep -v Warn | head -14 > gpurun_out/timeline_at.log
LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 3 > gpurun_out/e2e_at.log 2>&1
