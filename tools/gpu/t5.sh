# config-5 chunk stage times (+ optional pytest selection in $TESTS)
mkdir -p gpurun_out
python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5_${TAG:-x}.json 2>&1
cut -c1-400 gpurun_out/t5_${TAG:-x}.json
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest $TESTS -x -q -m gpu > gpurun_out/tests_${TAG:-x}.log 2>&1; echo tests rc $?; tail -3 gpurun_out/tests_${TAG:-x}.log; fi
