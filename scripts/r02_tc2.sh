mkdir -p gpurun_out
LCN_TCB_TRACE=1 LCN_TIMING=1 timeout 300 python scripts/probe.py c3 0.1 1 > gpurun_out/trace.log 2>&1; echo RC $? >> gpurun_out/trace.log
for parts in 7 1 2 4 0; do LCN_TC_PARTS=$parts timeout 300 python tests/parity_c3_gpu.py gpurun_out/parity_s005_p$parts.npz 0.005 > gpurun_out/parity_s005_p$parts.log 2>&1; done
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/probe_tc.log 2>&1; echo RC $? >> gpurun_out/probe_tc.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_tc.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_tc.log
