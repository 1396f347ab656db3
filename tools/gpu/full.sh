# full round-end style validation: gpu tests, smoke, both bench arms
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/full_tests.log 2>&1; echo tests rc $?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo smoke rc $?
timeout 900 python bench.py --impl reference > gpurun_out/full_bench_ref.log 2>&1; echo ref rc $?
timeout 900 python bench.py > gpurun_out/full_bench.log 2>&1; echo bench rc $?
tail -3 gpurun_out/full_tests.log; tail -2 gpurun_out/full_smoke.log; tail -c 600 gpurun_out/full_bench_ref.log; tail -c 1500 gpurun_out/full_bench.log
