# TC filter: cluster 4 (default) vs 2 vs 1
mkdir -p gpurun_out
for v in c4 c2 c1; do
  lib=paper_2107_06876_b200/_build/liblcn_b200.so; [ $v != c4 ] && lib=paper_2107_06876_b200/_build/liblcn_b200_$v.so
  LCN_LIB_PATH=$PWD/$lib timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum --clock-control none -k regex:assign_filter_tc -c 2 --csv python scripts/tc_bench.py 2000000 4096 0 > gpurun_out/tc_ap_$v.csv 2>&1
done
