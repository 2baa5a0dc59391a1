mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tcb_|band_tile|dense_tile" --csv --log-file gpurun_out/tc_launches.csv python scripts/probe.py c3 0.1 1 > gpurun_out/tc_launches.log 2>&1; echo RC $? >> gpurun_out/tc_launches.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tcb_kernel" -c 3 -o gpurun_out/prof_tcb -f python scripts/probe.py c3 0.1 1 > gpurun_out/prof_tcb.log 2>&1; echo RC $? >> gpurun_out/prof_tcb.log
