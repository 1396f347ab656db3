# round snapshot: smoke, full GPU suite, default bench, reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo gputest rc $?; tail -2 gpurun_out/gputest.log
S=$(date +%s); python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench rc $? wall $(( $(date +%s) - S )) s
tail -c 400 gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref rc $?
tail -c 800 gpurun_out/bench_ref.log
