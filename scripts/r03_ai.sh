mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "schedules" > gpurun_out/tests_ai.log 2>&1; echo TESTS $? >> gpurun_out/tests_ai.log
