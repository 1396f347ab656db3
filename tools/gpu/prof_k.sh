# ncu --set full of kernels matching $K on the config-5 chunk (one call)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -c ${C:-2} -o gpurun_out/prof_${TAG} -f python tools/time_coarse5.py --pairs 8 --once > gpurun_out/ncu_${TAG}.log 2>&1
echo rc $?
