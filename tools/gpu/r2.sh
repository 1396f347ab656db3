# config-5 profile: popc probe, launch list, ncu --set full of the chunk kernels
set -x
mkdir -p gpurun_out
nproc; lscpu | grep -m1 "Model name"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/popc_peak tools/diag/popc_peak.cu && /tmp/popc_peak > gpurun_out/popc.json 2>&1
python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches5.csv python tools/time_coarse5.py --pairs 8 --once > gpurun_out/ncu_ll.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_blur|k_lanczos|k_pyramid|k_fast_nms|k_measures|k_sel|k_select|k_orient|k_describe|k_match_jobs" -o gpurun_out/prof_r02a -f python tools/time_coarse5.py --pairs 8 --once > gpurun_out/ncu_full.log 2>&1
echo done
