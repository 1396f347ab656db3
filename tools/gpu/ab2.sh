# A/B: product library vs build/variants/$VAR.so on the config-5 chunk (+ tests on the product)
mkdir -p gpurun_out
for i in 1 2; do
XA_LIB_PATH=build/variants/${VAR:-old}.so python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/ab_${VAR:-old}_$i.json 2>&1
python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/ab_new_$i.json 2>&1
done
cat gpurun_out/ab_*.json
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest $TESTS -x -q -m gpu > gpurun_out/ab_tests.log 2>&1; echo tests rc $?; tail -3 gpurun_out/ab_tests.log; fi
