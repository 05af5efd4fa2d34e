mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_agg.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_agg.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_agg.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_agg.log').read().strip().splitlines()[-1]);print(d['value'], d['tflops_eq1'], d['roofline']['achieved'], d['clocks'], d['e2e'])"
