# ncu full + source of the TC assignment filter (one launch), csv pages only
mkdir -p gpurun_out /tmp/prof
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_filter_tc -s 1 -c 1 -o /tmp/prof/tc -f python scripts/tc_bench.py 2000000 4096 0 > gpurun_out/prof_tc_z.log 2>&1; echo RC $? >> gpurun_out/prof_tc_z.log
ncu -i /tmp/prof/tc.ncu-rep --page details --csv > gpurun_out/tc_z_details.csv 2>&1
ncu -i /tmp/prof/tc.ncu-rep --page source --csv --print-source sass > gpurun_out/tc_z_source.csv 2>&1
ls -la gpurun_out/tc_z_*
