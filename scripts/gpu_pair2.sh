mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "tensor_core" -p no:cacheprovider -x > gpurun_out/pytest_pair.log 2>&1; echo "tc tests rc=$?"; tail -2 gpurun_out/pytest_pair.log
for ch in 2 4; do
QSG_TC_CHUNK=$ch timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ch$ch.log 2>&1; echo "bench ch=$ch rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_ch$ch.log').read().strip().splitlines()[-1]);print(d['value'], d['tflops_eq1'], d['roofline']['achieved'], d['roofline']['kernel'], d['clocks'])"
done
QSG_TC_CHUNK=4 timeout 300 python scripts/tc_accuracy.py > gpurun_out/tc_ch4.log 2>&1; grep -E "'k': (16|65536)|rel_l2" gpurun_out/tc_ch4.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "all rc=$?"; tail -3 gpurun_out/pytest_gpu.log
