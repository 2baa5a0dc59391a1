# r02 session 2: state check after re-entry: GPU tests, bench, full C3 parity dump
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; free -g >> gpurun_out/host.txt; lscpu | grep -i "model name" >> gpurun_out/host.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo RC $? >> gpurun_out/bench.log
timeout 1200 python tests/parity_c3_gpu.py gpurun_out/parity_c3_gpu.npz 1.0 > gpurun_out/parity_c3.log 2>&1; echo RC $? >> gpurun_out/parity_c3.log
