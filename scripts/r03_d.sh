mkdir -p gpurun_out
for v in "LCN_PP_FILTER=f16" "LCN_PP_FILTER=i8"; do
  echo "== $v" >> gpurun_out/timeline_d.log
  env $v timeout 300 python scripts/timeline.py 2000000 4096 >> gpurun_out/timeline_d.log 2>&1
done
