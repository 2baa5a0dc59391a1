mkdir -p gpurun_out
LCN_TILE_DEBUG=1 LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 1 > gpurun_out/e2e_aw.log 2>&1
LCN_LLOYD_TILE_ORDER=0 LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 1 >> gpurun_out/e2e_aw.log 2>&1
