# exact-pass variants (no PDL timelines: kernel durations)
mkdir -p gpurun_out
for v in "LCN_PP_EXACT=smem" "LCN_PP_EXACT_CTAS=1" "LCN_PP_EXACT=lane"; do
  echo "== $v" >> gpurun_out/timeline_j.log
  env $v LCN_PP_PDL=0 timeout 300 python scripts/timeline.py 2000000 4096 2>&1 | grep -v Warn | head -12 >> gpurun_out/timeline_j.log
done
