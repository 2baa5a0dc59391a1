# r02: dense anchor recomputed on tcgen05 (parity) + probe timings at configs[2]
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dense_recompute or dense_anchor" > gpurun_out/dense_tc.log 2>&1; echo TESTS $? >> gpurun_out/dense_tc.log
