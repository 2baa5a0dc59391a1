mkdir -p gpurun_out
for v in 1 0 1 0; do
  echo "== LCN_SEED_PRIORITY=$v" >> gpurun_out/e2e_am.log
  LCN_SEED_PRIORITY=$v LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 3 2>&1 | grep -E "^rep|seeding \(" >> gpurun_out/e2e_am.log
done
