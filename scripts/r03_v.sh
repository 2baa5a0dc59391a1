# persistent fold_round, unstaged walk by default
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "kmeans_pp or lloyd or lsh_buckets" > gpurun_out/tests_v.log 2>&1; echo TESTS $? >> gpurun_out/tests_v.log
LCN_PP_WALK_STAGED=1 LCN_PP_CERT_SLACK=20000 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "kmeans_pp" >> gpurun_out/tests_v.log 2>&1; echo TESTS_STAGED $? >> gpurun_out/tests_v.log
LCN_TIMING=1 timeout 600 python scripts/e2e_host_probe.py 3 > gpurun_out/e2e_v.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pp_|seed_dist|fold_round" -s 6000 -c 70 --csv --log-file gpurun_out/launches_seed_v.csv python scripts/km_one.py > gpurun_out/ncu_list_seed_v.log 2>&1
