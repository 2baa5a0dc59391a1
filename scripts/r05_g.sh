# intermittent bench stall, second pass: short bench runs (no e2e) alternating band overlap on/off
mkdir -p gpurun_out
: > gpurun_out/stall_r05g.log
for rep in 1 2 3 4 5 6 7 8; do
for ov in 1 0; do
  s0=$SECONDS
  LCN_BAND_OVERLAP=$ov timeout -s ABRT 150 python -X faulthandler bench.py --no-e2e --no-cpu --no-c4 --no-dense --no-fp64 > gpurun_out/stallg_${ov}_${rep}.log 2> gpurun_out/stallg_${ov}_${rep}.err
  rc=$?
  echo "overlap=$ov rep=$rep rc=$rc wall=$((SECONDS - s0)) $(python -c "
import json
try:
    d=json.loads(open('gpurun_out/stallg_${ov}_${rep}.log').read().strip().splitlines()[-1]); print('value',round(d['value'],1),'build_s',round(d['build_s'],3))
except Exception as e: print('noline')
")" >> gpurun_out/stall_r05g.log
done; done
