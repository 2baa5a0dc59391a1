# r02: launch list of the k-means++ seeding kernels (steady state) at configs[3]
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pp_|fold_|seed_dist" -s 6000 -c 200 --csv --log-file gpurun_out/seed_launches.csv python scripts/probe.py c3 1.0 1 > gpurun_out/seed_launches.log 2>&1; echo RC $? >> gpurun_out/seed_launches.log
