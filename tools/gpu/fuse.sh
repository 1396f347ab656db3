# fused ORB levels in the Lanczos resampler: A/B on the config-5 chunk + parity tests
mkdir -p gpurun_out
XA_LZ_FUSE=0 python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5_fuse0.json 2>&1
XA_LZ_FUSE=1 python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5_fuse1.json 2>&1
XA_LIB_PATH=build/variants/fc3.so python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/t5_fuse1_fc3.json 2>&1
cat gpurun_out/t5_fuse0.json gpurun_out/t5_fuse1.json gpurun_out/t5_fuse1_fc3.json | tail -c 1500
if [ -n "$TESTS" ]; then
timeout 1200 python -m pytest $TESTS -x -q -m gpu > gpurun_out/fuse_tests.log 2>&1
echo tests rc $?; tail -3 gpurun_out/fuse_tests.log
fi
