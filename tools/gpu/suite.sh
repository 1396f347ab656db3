# smoke + full GPU suite (the driver's round-end checks)
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo gputest rc $?; tail -3 gpurun_out/gputest.log
