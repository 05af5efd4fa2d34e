mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "tensor_core" -p no:cacheprovider -x > gpurun_out/pytest_pers.log 2>&1; echo "tc tests rc=$?"; tail -2 gpurun_out/pytest_pers.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pers.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_pers.log').read().strip().splitlines()[-1]);print(d['value'], d['tflops_eq1'], d['roofline']['achieved'], d['roofline']['kernel'], d['clocks'])"
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/plain3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv $CMD > gpurun_out/ncu_launch3.log 2>&1; echo "ncu list rc=$?"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "all rc=$?"; tail -3 gpurun_out/pytest_gpu.log
