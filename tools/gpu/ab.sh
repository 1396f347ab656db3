# A/B of Lanczos run lengths on the config-5 chunk + the view/coarse parity tests
mkdir -p gpurun_out
for r in 1 2 3; do XA_LZ_RUN_MAX=$r python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5_run$r.json 2>&1; done
timeout 900 python -m pytest tests/test_gpu_views.py tests/test_gpu_coarse.py tests/test_gpu_pinned.py tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/views_tests.log 2>&1
echo tests rc $?
cat gpurun_out/t5_run*.json; tail -3 gpurun_out/views_tests.log
