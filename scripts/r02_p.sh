# r02: sparse-only operator band kernels with fp32 exponents: parity tests + configs[3] timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -k "sparse or bp or support or dense_anchor or lsh_schemes" > gpurun_out/tests_p.log 2>&1; echo TESTS $? >> gpurun_out/tests_p.log
PROBE_SPARSE=1 timeout 300 python scripts/probe.py c3 1.0 2 > gpurun_out/probe_sparse_p.log 2>&1; echo RC $? >> gpurun_out/probe_sparse_p.log
