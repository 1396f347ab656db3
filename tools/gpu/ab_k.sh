mkdir -p gpurun_out
python tools/time_coarse5.py --pairs 64 --steps 3 --noprof > gpurun_out/k8.json 2>&1
XA_BATCH_PAIRS=16 python tools/time_coarse5.py --pairs 64 --steps 3 --noprof > gpurun_out/k16.json 2>&1
XA_BATCH_PAIRS=4 python tools/time_coarse5.py --pairs 64 --steps 3 --noprof > gpurun_out/k4.json 2>&1
for f in gpurun_out/k*.json; do echo $f; cat $f; done
