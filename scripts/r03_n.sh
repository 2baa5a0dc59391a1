mkdir -p gpurun_out
LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 2 > gpurun_out/e2e_n.log 2>&1; echo RC $? >> gpurun_out/e2e_n.log
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/timing_n.log 2>&1
