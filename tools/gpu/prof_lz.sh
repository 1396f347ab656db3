mkdir -p gpurun_out
XA_LZ_RUN_MAX=${RUNMAX:-3} timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lanczos" -o gpurun_out/prof_${TAG:-lz} -f python tools/time_coarse5.py --pairs 8 --once > gpurun_out/ncu_${TAG:-lz}.log 2>&1
echo rc $?
