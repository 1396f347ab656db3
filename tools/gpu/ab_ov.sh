mkdir -p gpurun_out
for i in 1 2; do
XA_OVERLAP=0 python tools/time_coarse5.py --pairs 16 --steps 3 --noprof > gpurun_out/ov_off_$i.json 2>&1
python tools/time_coarse5.py --pairs 16 --steps 3 --noprof > gpurun_out/ov_on_$i.json 2>&1
done
for f in gpurun_out/ov_*.json; do echo $f; cat $f; done
timeout 1500 python -m pytest tests/test_gpu_batch.py tests/test_gpu_coarse.py tests/test_gpu_configs.py tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/ov_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/ov_tests.log
ARGS="--no-secondary --no-cpu-baseline" bash tools/gpu/bench_only.sh
python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench.log') if l.startswith('{')][-1]); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['stage_ms'], d['results'])"
