# tensor-core Hamming matcher vs XOR+POPC: config-4 timing/digest, config-5 chunk, tests
mkdir -p gpurun_out
python tools/time_cfg4.py 5 > gpurun_out/cfg4_tc.json 2>&1; cat gpurun_out/cfg4_tc.json
XA_MATCH_TC=0 python tools/time_cfg4.py 3 > gpurun_out/cfg4_popc.json 2>&1; cat gpurun_out/cfg4_popc.json
python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5_tc.json 2>&1; cut -c1-330 gpurun_out/t5_tc.json; echo
XA_MATCH_TC=0 python tools/time_coarse5.py --pairs 8 --steps 3 > gpurun_out/t5_popc.json 2>&1; cut -c1-330 gpurun_out/t5_popc.json; echo
timeout 1200 python -m pytest tests/test_gpu_match.py tests/test_gpu_kats.py tests/test_gpu_pinned.py tests/test_gpu_coarse.py -x -q -m gpu > gpurun_out/tests_tc.log 2>&1; echo tests rc $?; tail -3 gpurun_out/tests_tc.log
