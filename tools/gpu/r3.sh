# config-3 / config-4 ncu captures + a 2-rank bench run (gloo collectives, one GPU) for the N>1 path
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_blur|k_lanczos" -o gpurun_out/prof_r02_cfg3 -f python tools/run_cfg.py cfg3 > gpurun_out/ncu_cfg3.log 2>&1; echo cfg3 rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_match" -o gpurun_out/prof_r02_cfg4 -f python tools/run_cfg.py cfg4 > gpurun_out/ncu_cfg4.log 2>&1; echo cfg4 rc $?
XA_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-secondary > gpurun_out/bench_n2.log 2>&1; echo n2 rc $?
tail -c 1500 gpurun_out/bench_n2.log
