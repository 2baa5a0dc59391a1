# Sparse-only operator with the single-read online log-sum-exp consumer: parity tests, timing, one ncu capture.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "sparse or bp or staged or integration or panel" > gpurun_out/t_r05b.log 2>&1; echo TESTS $? >> gpurun_out/t_r05b.log
PROBE_SPARSE=1 timeout 600 python scripts/probe.py c3 1.0 3 > gpurun_out/sparse_r05b.log 2>&1; echo PROBE $? >> gpurun_out/sparse_r05b.log
PROBE_SPARSE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_stream_kernel --launch-skip 40 --launch-count 2 -o gpurun_out/prof_sparse_lse_r05b -f python scripts/probe.py c3 1.0 1 > gpurun_out/ncu_sparse_r05b.log 2>&1; echo NCU $? >> gpurun_out/ncu_sparse_r05b.log
