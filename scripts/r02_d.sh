# r02: band_stream_kernel claim-ahead: correctness + C3 timing
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "band or lcn or split or wide" > gpurun_out/band_tests.log 2>&1; echo TESTS $? >> gpurun_out/band_tests.log
timeout 300 python scripts/probe.py c3 1.0 3 > gpurun_out/probe_d.log 2>&1; echo RC $? >> gpurun_out/probe_d.log
