mkdir -p gpurun_out
timeout 300 python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/abt_base.json 2>&1; echo base; cut -c1-330 gpurun_out/abt_base.json; echo
for v in $VARIANTS; do XA_LIB_PATH=build/variants/$v.so timeout 300 python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/abt_$v.json 2>&1; echo $v; cut -c1-330 gpurun_out/abt_$v.json; echo; done
