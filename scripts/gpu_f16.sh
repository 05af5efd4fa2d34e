mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_f16_kernels.log 2>&1; rc=$?; echo "kernels rc=$rc"; tail -15 gpurun_out/pytest_f16_kernels.log
[ $rc -eq 0 ] || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_f16.log 2>&1; echo "all rc=$?"; tail -5 gpurun_out/pytest_f16.log
timeout 300 python scripts/tc_accuracy.py > gpurun_out/tc_f16.log 2>&1; echo "acc rc=$?"; cat gpurun_out/tc_f16.log
for v in f16 tf32; do
QSG_TC_PREC=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_f16_$v.log 2>&1; echo "bench f16=$v rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_f16_$v.log').read().strip().splitlines()[-1]);print(d['value'], d['tflops_eq1'], d['roofline']['achieved'], d['clocks'])"
done
