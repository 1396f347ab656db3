# A/B of the paired Lanczos path on the config-5 chunk + view/coarse parity tests
mkdir -p gpurun_out
XA_LZ_PAIR=0 python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5_pair0.json 2>&1
XA_LZ_PAIR=1 python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5_pair1.json 2>&1
XA_LIB_PATH=build/variants/lz2.so python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5_pair1_lz2.json 2>&1
timeout 900 python -m pytest tests/test_gpu_views.py tests/test_gpu_coarse.py tests/test_gpu_pinned.py tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/views_tests.log 2>&1
echo tests rc $?
cat gpurun_out/t5_pair*.json; tail -3 gpurun_out/views_tests.log
