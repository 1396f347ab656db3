mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${K:-k_match_tc}" -c ${C:-1} -o gpurun_out/prof_${TAG:-cfg4tc} -f python tools/run_cfg.py cfg4 > gpurun_out/ncu_${TAG:-cfg4tc}.log 2>&1
echo rc $?
