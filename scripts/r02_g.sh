# r02: the reference's unit tests through the drop-in shim on the B200
mkdir -p gpurun_out
timeout 1200 integration/_build/ref_tests_gpu > gpurun_out/shim_tests.log 2>&1; echo RC $? >> gpurun_out/shim_tests.log
