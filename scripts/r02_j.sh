# r02: the full-size configs[3] reference pipeline on the GPU box's host cores
# (GPU bucket ids + reference landmarks from this container), build-phase
# timing of our build (LCN_TIMING)
mkdir -p gpurun_out
nproc > gpurun_out/host_j.txt
LCN_TIMING=1 PROBE_BUILDS=2 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/timing_j.log 2>&1; echo RC $? >> gpurun_out/timing_j.log
LCN_REF_BLOCKED_CORRECTION=1 OMP_NUM_THREADS=$(nproc) timeout 3000 python oracle/parity_c3.py pipeline --scratch parity_in --ids parity_in/parity_c3_gpu.npz > gpurun_out/pipeline_box.log 2>&1; echo RC $? >> gpurun_out/pipeline_box.log
cp parity_in/ref_pipeline.json gpurun_out/ref_pipeline_box.json 2>/dev/null
