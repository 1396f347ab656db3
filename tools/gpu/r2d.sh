# round-2 final evidence: chunk + 64-pair stage times, bench, launch lists (chunk + bench), ncu --set full of the chunk kernels
mkdir -p gpurun_out
python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5_r2d.json 2>&1; cut -c1-600 gpurun_out/t5_r2d.json
python tools/time_coarse5.py --pairs 64 --steps 3 > gpurun_out/t5_r2d_64.json 2>&1; cut -c1-600 gpurun_out/t5_r2d_64.json
timeout 900 python bench.py > gpurun_out/bench_r2d.log 2>&1; echo bench rc $?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2d.csv python tools/time_coarse5.py --pairs 8 --once > gpurun_out/ncu_ll.log 2>&1; echo ll rc $?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2d_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary > gpurun_out/ncu_ll_bench.log 2>&1; echo llb rc $?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_blur|k_lanczos|k_pyramid|k_fast_nms|k_measures|k_sel|k_select|k_orient|k_describe|k_desc_pm1|k_match_umma|k_lanczos_sep" -o gpurun_out/prof_r02d -f python tools/time_coarse5.py --pairs 8 --once > gpurun_out/ncu_full.log 2>&1; echo full rc $?
