mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "all rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1b.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_r1b.log').read().strip().splitlines()[-1]);print(d['value'], d['tflops_eq1'], d['roofline']['achieved'], d['roofline']['kernel'], d['clocks'], d['cpu_baseline']['value'], d['e2e']['value'])"
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/plain4.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches4.csv $CMD > gpurun_out/ncu_launch4.log 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cgemm_tc2 -s 20 -c 1 -o gpurun_out/prof_tc2_s026 $CMD > gpurun_out/ncu_tc2b.log 2>&1; echo "ncu tc2 rc=$?"
