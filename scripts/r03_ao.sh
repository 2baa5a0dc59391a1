# TC filter ring: 6 stages of 32 features (default) vs 3 of 64
mkdir -p gpurun_out
for v in k32 k64; do
  lib=paper_2107_06876_b200/_build/liblcn_b200.so; [ $v = k64 ] && lib=paper_2107_06876_b200/_build/liblcn_b200_k64.so
  LCN_LIB_PATH=$PWD/$lib timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:assign_filter_tc -c 2 --csv python scripts/tc_bench.py 2000000 4096 0 > gpurun_out/tc_ao_$v.csv 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "assign or lloyd or lsh" > gpurun_out/tests_ao.log 2>&1; echo TESTS $? >> gpurun_out/tests_ao.log
