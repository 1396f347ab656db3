# A/B of an env switch ($ENVAB, e.g. XA_L0U8=0) on the config-5 chunk, same library
mkdir -p gpurun_out
for i in 1 2; do
env $ENVAB python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/abenv_off_$i.json 2>&1
python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/abenv_on_$i.json 2>&1
done
for f in gpurun_out/abenv_*.json; do echo $f; cat $f; done
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest $TESTS -x -q -m gpu > gpurun_out/abenv_tests.log 2>&1; echo tests rc $?; tail -3 gpurun_out/abenv_tests.log; fi
