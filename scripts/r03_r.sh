mkdir -p gpurun_out
LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 3 > gpurun_out/e2e_r.log 2>&1
