# Per setting: bench value + DRAM bytes / duration of the s026 launch (ncu, metrics only).
# SWEEP="A=1,B=2;A=2"
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
IFS=';' read -ra RUNS <<< "$SWEEP"
i=0
for r in "${RUNS[@]}"; do
  envs=$(echo "$r" | tr ',' ' ')
  env $envs timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/dsweep_$i.log 2>&1
  echo "[$r] rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/dsweep_$i.log').read().strip().splitlines()[-1]);print('   ', round(d['value'],1), round(d['tflops_eq1'],1), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  env $envs timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:cgemm_f16_pair -s ${IDX:-20} -c 1 $CMD 2>&1 | grep -E "gpu__time|dram__bytes|hit_rate|tensor_cycles" | sed 's/^/    /'
  i=$((i+1))
done
