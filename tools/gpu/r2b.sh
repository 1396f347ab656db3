# round-2 evidence: chunk stage times, launch lists (chunk + bench), ncu --set full of the chunk kernels, bench
mkdir -p gpurun_out
python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5_r2c.json 2>&1; cut -c1-400 gpurun_out/t5_r2c.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2c.csv python tools/time_coarse5.py --pairs 8 --once > gpurun_out/ncu_ll.log 2>&1; echo ll rc $?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_blur|k_lanczos|k_pyramid|k_fast_nms|k_measures|k_sel|k_select|k_orient|k_describe|k_desc_pm1|k_match_umma|k_lanczos_sep" -o gpurun_out/prof_r02c -f python tools/time_coarse5.py --pairs 8 --once > gpurun_out/ncu_full.log 2>&1; echo full rc $?


