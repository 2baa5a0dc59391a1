# ncu of the split seeding chain kernels (early / late steps); csv pages only
mkdir -p gpurun_out /tmp/prof
export LCN_PP_CHUNK=0
for w in "early 1200" "late 12000"; do
  set -- $w
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pp_filter_kernel|pp_prune_kernel|pp_exact_kernel|pp_pick_kernel" -s $2 -c 4 -o /tmp/prof/seed_$1 -f python scripts/km_one.py > gpurun_out/prof_seed_h_$1.log 2>&1; echo RC $? >> gpurun_out/prof_seed_h_$1.log
  ncu -i /tmp/prof/seed_$1.ncu-rep --page details --csv > gpurun_out/seed_$1_details.csv 2>&1
  ncu -i /tmp/prof/seed_$1.ncu-rep --page raw --csv > gpurun_out/seed_$1_raw.csv 2>&1
done
ls -la gpurun_out/
