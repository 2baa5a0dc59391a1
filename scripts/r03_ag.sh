# single-pass online LSE in the band kernel (sparse-only operator)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bp.py tests/test_gpu_staged.py -q -x -k "sparse or config0 or lsh_schemes or bp" > gpurun_out/tests_ag.log 2>&1; echo TESTS $? >> gpurun_out/tests_ag.log
PROBE_SPARSE=1 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/sp_ag_timing.log 2>&1
