# Bench the default config under several env settings: SWEEP="A=1,B=2;A=2" (';' separates runs).
mkdir -p gpurun_out
IFS=';' read -ra RUNS <<< "$SWEEP"
i=0
for r in "${RUNS[@]}"; do
  envs=$(echo "$r" | tr ',' ' ')
  env $envs timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline $BENCH_ARGS > gpurun_out/sweep_$i.log 2>&1
  echo "[$r] rc=$? $(grep -h 'co-resident' gpurun_out/sweep_$i.log | sort -u | tr '\n' ' ')"
  python -c "import json;d=json.loads(open('gpurun_out/sweep_$i.log').read().strip().splitlines()[-1]);print('   ', round(d['value'],1), round(d['tflops_eq1'],1), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  i=$((i+1))
done
