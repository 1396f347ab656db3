# full round-end style validation: gpu tests, smoke, both bench arms
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/full_tests.log 2>&1; echo tests rc $?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo smoke rc $?
timeout 900 python bench.py --impl reference > gpurun_out/full_bench_ref.log 2>&1; echo ref rc $?
timeout 900 python bench.py > gpurun_out/full_bench.log 2>&1; echo bench rc $?
tail -3 gpurun_out/full_tests.log; tail -2 gpurun_out/full_smoke.log; tail -c 600 gpurun_out/full_bench_ref.log; tail -c 1500 gpurun_out/full_bench.log
# 2 ranks on this one GPU (gloo collectives): the sharded bench path end to end; same counts digest as 1 rank
XA_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/full_bench_2rank.log 2>&1; echo 2rank rc $?
grep -o '"counts_sha256_16": "[0-9a-f]*"' gpurun_out/full_bench.log gpurun_out/full_bench_2rank.log
grep -o '"n_gpus": [0-9]*, "steps": [0-9]*' gpurun_out/full_bench_2rank.log
