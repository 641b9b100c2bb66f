python tools/diag_knn.py 2>&1 | tail -30
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_r01.csv python tools/profile_c2.py 12 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tag_env_kernel -s 6 -c 1 -o gpurun_out/prof_c2_v1 python tools/profile_c2.py 8 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
