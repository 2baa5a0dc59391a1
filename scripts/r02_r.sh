# r02: ncu of one early and one late k-means++ filter launch at configs[3] (stall sites)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pp_filter_exact -s 600 -c 1 -o gpurun_out/prof_filter_early -f python scripts/probe.py c3 1.0 1 > gpurun_out/prof_filter_early.log 2>&1; echo RC $? >> gpurun_out/prof_filter_early.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pp_filter_exact -s 6000 -c 1 -o gpurun_out/prof_filter_late -f python scripts/probe.py c3 1.0 1 > gpurun_out/prof_filter_late.log 2>&1; echo RC $? >> gpurun_out/prof_filter_late.log
