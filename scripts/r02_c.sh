# r02: ncu --set full of the band_stream_kernel launches of one configs[3] iteration (source-level stalls)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_stream_kernel -s 8 -c 4 -o gpurun_out/prof_band_r02 -f python scripts/probe.py c3 1.0 1 > gpurun_out/prof_band_r02.log 2>&1; echo RC $? >> gpurun_out/prof_band_r02.log
