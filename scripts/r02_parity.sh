# r02: GPU tests + full-size configs[3] parity dump (GPU half).
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; free -g >> gpurun_out/host.txt; lscpu | grep -i "model name" >> gpurun_out/host.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo TESTS $? >> gpurun_out/gpu_tests.log
timeout 300 python tests/parity_c3_gpu.py gpurun_out/parity_s005.npz 0.005 > gpurun_out/parity_s005.log 2>&1; echo RC $? >> gpurun_out/parity_s005.log
timeout 1200 python tests/parity_c3_gpu.py gpurun_out/parity_c3_gpu.npz 1.0 > gpurun_out/parity_c3.log 2>&1; echo RC $? >> gpurun_out/parity_c3.log
