mkdir -p gpurun_out
S=$(date +%s); python bench.py ${ARGS} > gpurun_out/bench${TAG}.log 2> gpurun_out/bench${TAG}.err; echo bench rc $? wall $(( $(date +%s) - S )) s
tail -c 300 gpurun_out/bench${TAG}.err
