# ncu --set full of k_lanczos_smem, single vs pair mode (config-5 chunk)
mkdir -p gpurun_out
for m in 0 1; do
XA_LZ_PAIR=$m timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanczos_smem -c 1 -o gpurun_out/prof_lzp$m -f python tools/time_coarse5.py --pairs 8 --once > gpurun_out/ncu_lzp$m.log 2>&1
echo rc $?
done
