# Tests + default bench line (+ optional extra bench args via BENCH_ARGS).
mkdir -p gpurun_out
TAG=${TAG:-check}
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_${TAG}_kernels.log 2>&1; rc=$?; echo "kernels rc=$rc"; tail -15 gpurun_out/pytest_${TAG}_kernels.log
[ $rc -eq 0 ] || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1; echo "all rc=$?"; tail -5 gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline $BENCH_ARGS > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_${TAG}.log').read().strip().splitlines()[-1]);print(d['value'], d['tflops_eq1'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['kernel'], d['e2e']['value'], d['clocks'])"
