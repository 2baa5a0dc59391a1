# ncu of the sparse-only operator's LSE band pass (source-level), csv pages only
mkdir -p gpurun_out /tmp/prof
PROBE_SPARSE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_stream -s 4 -c 1 -o /tmp/prof/sp -f python scripts/probe.py c3 1.0 1 > gpurun_out/prof_sp_ad.log 2>&1; echo RC $? >> gpurun_out/prof_sp_ad.log
ncu -i /tmp/prof/sp.ncu-rep --page details --csv > gpurun_out/sp_ad_details.csv 2>&1
ncu -i /tmp/prof/sp.ncu-rep --page source --csv --print-source sass > gpurun_out/sp_ad_source.csv 2>&1
PROBE_SPARSE=1 timeout 300 python scripts/probe.py c3 1.0 1 > gpurun_out/sp_ad_timing.log 2>&1
