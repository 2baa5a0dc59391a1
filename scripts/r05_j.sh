# clean-built library: smoke; then a longer soak of LCN_BAND_OVERLAP=2 (40 short bench runs, 150 s timeout each)
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py > gpurun_out/smoke_r05j.log 2>&1; echo SMOKE $? >> gpurun_out/smoke_r05j.log
: > gpurun_out/stall_r05j.log
for rep in $(seq 1 40); do
  s0=$SECONDS
  LCN_BAND_OVERLAP=2 timeout -s ABRT 150 python -X faulthandler bench.py --no-e2e --no-cpu --no-c4 --no-dense --no-fp64 > gpurun_out/stallj_${rep}.log 2> gpurun_out/stallj_${rep}.err
  echo "overlap=2 rep=$rep rc=$? wall=$((SECONDS - s0))" >> gpurun_out/stall_r05j.log
done
