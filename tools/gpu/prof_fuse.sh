mkdir -p gpurun_out
for f in 0 1; do
XA_LZ_FUSE=$f timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanczos_smem -c 1 -o gpurun_out/prof_fuse$f -f python tools/time_coarse5.py --pairs 8 --once > gpurun_out/ncu_fuse$f.log 2>&1
echo rc $?
done
