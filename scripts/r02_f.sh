# r02: staged drop-in API vs the reference's stages
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_staged.py -q -x > gpurun_out/staged.log 2>&1; echo TESTS $? >> gpurun_out/staged.log
