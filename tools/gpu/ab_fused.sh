mkdir -p gpurun_out
for v in $VARIANTS; do XA_LIB_PATH=build/variants/$v.so python tools/time_coarse5.py --pairs 8 --steps 3 > gpurun_out/ab_$v.json 2>&1; done
for v in $VARIANTS; do echo $v; cut -c1-130 gpurun_out/ab_$v.json; done
