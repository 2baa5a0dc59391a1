# intermittent bench stall: repeated short bench runs with band overlap on/off, traceback dump on timeout
mkdir -p gpurun_out
: > gpurun_out/stall_r05f.log
for rep in 1 2 3 4; do
for ov in 1 0; do
  t0=$(date +%s.%N)
  LCN_BAND_OVERLAP=$ov timeout -s ABRT 240 python -X faulthandler bench.py --no-cpu --no-c4 --no-dense --no-fp64 > gpurun_out/stall_${ov}_${rep}.log 2> gpurun_out/stall_${ov}_${rep}.err
  rc=$?
  t1=$(date +%s.%N)
  echo "overlap=$ov rep=$rep rc=$rc wall=$(echo "$t1 - $t0" | bc) $(python -c "
import json,sys
try:
    d=json.loads(open('gpurun_out/stall_${ov}_${rep}.log').read().strip().splitlines()[-1]); print('value',round(d['value'],1),'e2e_s',round(d['e2e']['solve_s'],3))
except Exception as e: print('noline')
")" >> gpurun_out/stall_r05f.log
done; done
