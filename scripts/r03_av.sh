# Lloyd tile skipping with grouped centroid tiles
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -k "lloyd or assign or lsh or kmeans or shard or lcn_small or schedules" > gpurun_out/tests_av.log 2>&1; echo TESTS $? >> gpurun_out/tests_av.log
for v in 1 0; do
  echo "== LCN_LLOYD_TILE_ORDER=$v" >> gpurun_out/e2e_av.log
  LCN_LLOYD_TILE_ORDER=$v LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 3 2>&1 | grep -E "^rep|lsh k-means|tile skipping" >> gpurun_out/e2e_av.log
done
