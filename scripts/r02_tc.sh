# r02: tensor-core build check: GPU tests, C3 build timings (TC vs exact tiles), parity dump s005 in TC mode
mkdir -p gpurun_out
timeout 300 python tests/parity_c3_gpu.py gpurun_out/parity_s005_tc.npz 0.005 > gpurun_out/parity_s005_tc.log 2>&1; echo RC $? >> gpurun_out/parity_s005_tc.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_tc.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests_tc.log
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/probe_tc.log 2>&1; echo RC $? >> gpurun_out/probe_tc.log
LCN_EXACT_BUILD=1 LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/probe_exact.log 2>&1; echo RC $? >> gpurun_out/probe_exact.log
