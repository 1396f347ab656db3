# time_coarse5 (config-5 chunk) for the product library and build/variants/$VARIANTS
mkdir -p gpurun_out
python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/ab_base.json 2>&1
for v in $VARIANTS; do XA_LIB_PATH=build/variants/$v.so python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/ab_$v.json 2>&1; done
for f in gpurun_out/ab_*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['ms_step'], d['stages'], d['counts_sha16'], d['sum_counts'])" 2>&1 | tail -1; done
