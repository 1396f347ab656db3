# tcgen05 matcher: config-4 digest/timing vs the IMMA and POPC kernels, config-5 chunk, tests
mkdir -p gpurun_out
timeout 120 python tools/time_cfg4.py 5 > gpurun_out/cfg4_umma.json 2>&1; echo "rc $?"; tail -3 gpurun_out/cfg4_umma.json
XA_MATCH_UMMA=0 timeout 120 python tools/time_cfg4.py 3 > gpurun_out/cfg4_imma.json 2>&1; cat gpurun_out/cfg4_imma.json
timeout 120 python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5_umma.json 2>&1; echo "rc $?"; tail -c 400 gpurun_out/t5_umma.json; echo
if [ -n "$TESTS" ]; then timeout 900 python -m pytest $TESTS -x -q -m gpu > gpurun_out/tests_umma.log 2>&1; echo tests rc $?; tail -3 gpurun_out/tests_umma.log; fi
