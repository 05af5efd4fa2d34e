# GPU tests + bench lines for configs 2 (default), 4 and 5.  TAG names the logs.
mkdir -p gpurun_out
TAG=${TAG:-all}
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_${TAG}.log
for c in 2 4 5; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c$c.log 2>&1; echo "c$c rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/bench_${TAG}_c$c.log').read().strip().splitlines()[-1]);print('   ', d['value'], round(d['tflops_eq1'],1), round(d['roofline']['achieved'],1), round(d['roofline']['frac'],3), d['roofline']['kernel'], round(d['e2e']['value'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
