mkdir -p gpurun_out
LCN_TCB_TRACE=1 LCN_TIMING=1 timeout 300 python scripts/probe.py c3 0.1 1 > gpurun_out/trace.log 2>&1; echo RC $? >> gpurun_out/trace.log
