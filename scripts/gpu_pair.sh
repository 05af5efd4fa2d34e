mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "tensor_core" -p no:cacheprovider -x > gpurun_out/pytest_pair.log 2>&1; echo "tc tests rc=$?"; tail -5 gpurun_out/pytest_pair.log
timeout 300 python scripts/tc_accuracy.py > gpurun_out/tc_pair.log 2>&1; echo "acc rc=$?"; grep -E "'k': (16|1024|65536)|rel_l2" gpurun_out/tc_pair.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pair.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_pair.log').read().strip().splitlines()[-1]);print(d['value'], d['tflops_eq1'], d['roofline']['achieved'], d['roofline']['kernel'], d['clocks'])"
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "all rc=$?"; tail -3 gpurun_out/pytest_gpu.log
