# config-5 chunk timing under each env setting in $ENVS (";"-separated)
mkdir -p gpurun_out
IFS=';' read -ra E <<< "$ENVS"
i=0
for e in "${E[@]}"; do env $e python tools/time_coarse5.py --pairs 8 --steps 5 > gpurun_out/abenv_$i.json 2>&1; echo "[$e]"; cut -c1-240 gpurun_out/abenv_$i.json; echo; i=$((i+1)); done
