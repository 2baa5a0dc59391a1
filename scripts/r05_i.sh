# Soak of LCN_BAND_OVERLAP=2 (overlapping band triggers its dependent only by exiting): short bench runs, 150 s timeout each;
# then the default path once more after the rebuild (band tests + bench).
mkdir -p gpurun_out
: > gpurun_out/stall_r05i.log
for rep in $(seq 1 24); do
  s0=$SECONDS
  LCN_BAND_OVERLAP=2 timeout -s ABRT 150 python -X faulthandler bench.py --no-e2e --no-cpu --no-c4 --no-dense --no-fp64 > gpurun_out/stalli_${rep}.log 2> gpurun_out/stalli_${rep}.err
  rc=$?
  echo "overlap=2 rep=$rep rc=$rc wall=$((SECONDS - s0)) $(python -c "
import json
try:
    d=json.loads(open('gpurun_out/stalli_${rep}.log').read().strip().splitlines()[-1]); print('value',round(d['value'],1))
except Exception as e: print('noline')
")" >> gpurun_out/stall_r05i.log
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "lcn or band or panel or static" > gpurun_out/t_r05i.log 2>&1; echo TESTS $? >> gpurun_out/t_r05i.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_r05i.log 2> gpurun_out/bench_r05i.err; echo BENCH $? >> gpurun_out/bench_r05i.err
