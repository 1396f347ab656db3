mkdir -p gpurun_out
timeout 120 python tools/time_cfg4.py 7 > gpurun_out/c4_base.json 2>&1; echo base; cat gpurun_out/c4_base.json
for v in $VARIANTS; do XA_LIB_PATH=build/variants/$v.so timeout 120 python tools/time_cfg4.py 7 > gpurun_out/c4_$v.json 2>&1; echo $v; cat gpurun_out/c4_$v.json; done
