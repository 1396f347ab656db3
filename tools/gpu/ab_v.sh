# base vs build/variants/$V: config-5 chunk timing + $TESTS on the variant
mkdir -p gpurun_out
python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/ab_base.json 2>&1
XA_LIB_PATH=build/variants/$V.so python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/ab_$V.json 2>&1
cut -c1-330 gpurun_out/ab_base.json; echo; cut -c1-330 gpurun_out/ab_$V.json; echo
if [ -n "$TESTS" ]; then XA_LIB_PATH=build/variants/$V.so timeout 1500 python -m pytest $TESTS -x -q -m gpu > gpurun_out/tests_$V.log 2>&1; echo tests rc $?; tail -3 gpurun_out/tests_$V.log; fi
