# ncu (csv pages) of the current seeding chain kernels, early / late steps; single sequence (lloyd)
mkdir -p gpurun_out /tmp/prof
for w in "early 1200" "late 20000"; do
  set -- $w
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pp_filter_i8_kernel|pp_prune_kernel|pp_exact_kernel|pp_pick_kernel" -s $2 -c 4 -o /tmp/prof/seed_$1 -f python scripts/km_one.py > gpurun_out/prof_seed_u_$1.log 2>&1; echo RC $? >> gpurun_out/prof_seed_u_$1.log
  ncu -i /tmp/prof/seed_$1.ncu-rep --page details --csv > gpurun_out/seed_u_$1_details.csv 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"pp_|seed_dist|fold_round" -s 6000 -c 70 --csv --log-file gpurun_out/launches_seed_u.csv python scripts/km_one.py > gpurun_out/ncu_list_seed_u.log 2>&1; echo RC $? >> gpurun_out/ncu_list_seed_u.log
