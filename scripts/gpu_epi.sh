# Kernel tests + configs 3, 4, 2 with per-op profiles (epilogue / narrow-N changes).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -m gpu -q -x -p no:cacheprovider > gpurun_out/epi_pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/epi_pytest.log
for c in 3 4 2; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --profile-out gpurun_out/prof_ops_${TAG:-epi}_c$c.jsonl > gpurun_out/${TAG:-epi}_c$c.log 2>&1; echo "c$c rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/${TAG:-epi}_c$c.log').read().strip().splitlines()[-1]);print('   ', d['value'], round(d['tflops_eq1'],1), round(d['roofline']['achieved'],1), round(d['roofline']['frac'],3), d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
