# TC assignment filter: full 3xTF32 vs hi.hi only (feed- or MMA-bound?), cluster 4 vs 8
mkdir -p gpurun_out
for v in "c4 0" "c4 1" "c8 0" "c8 1"; do
  set -- $v
  lib=paper_2107_06876_b200/_build/liblcn_b200.so; [ $1 = c8 ] && lib=paper_2107_06876_b200/_build/liblcn_b200_c8.so
  LCN_LIB_PATH=$PWD/$lib timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum --clock-control none -k regex:assign_filter_tc -c 2 --csv python scripts/tc_bench.py 2000000 4096 $2 > gpurun_out/tc_y_$1_$2.csv 2>&1
done
