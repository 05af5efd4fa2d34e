# One bench line per config (N=1) with the current code -> gpurun_out/final_c*.log
mkdir -p gpurun_out
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-2} --warmup 2 --no-cpu-baseline > gpurun_out/final_c$c.log 2>&1; echo "c$c rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/final_c$c.log').read().strip().splitlines()[-1]);print('   ', d['value'], round(d['tflops_eq1'],1), round(d['roofline']['achieved'],1), round(d['roofline']['frac'],3), d['e2e']['value'], d['clocks']['sm_mhz'])"
done
