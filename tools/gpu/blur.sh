mkdir -p gpurun_out
XA_BLUR_RUNS=0 timeout 300 python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5_br0.json 2>&1; cut -c1-330 gpurun_out/t5_br0.json; echo
timeout 300 python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5_br1.json 2>&1; cut -c1-330 gpurun_out/t5_br1.json; echo
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest $TESTS -x -q -m gpu > gpurun_out/tests_blur.log 2>&1; echo tests rc $?; tail -5 gpurun_out/tests_blur.log; fi
