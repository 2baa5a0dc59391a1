# r02: ncu of the sparse-only row band kernel at configs[3]
mkdir -p gpurun_out
PROBE_SPARSE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_row_band -s 4 -c 1 -o gpurun_out/prof_sparse_y -f python scripts/probe.py c3 1.0 1 > gpurun_out/prof_sparse_y.log 2>&1; echo RC $? >> gpurun_out/prof_sparse_y.log
