mkdir -p gpurun_out
QSG_TC_RAWHI=1 timeout 600 python scripts/tc_accuracy.py > gpurun_out/tc_rawhi.log 2>&1; echo "rc=$?"; grep -E "'k': (16|1024|65536)|rel_l2" gpurun_out/tc_rawhi.log
QSG_TC_RAWHI=1 timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_rawhi.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_rawhi.log').read().strip().splitlines()[-1]);print(d['value'], d['tflops_eq1'], d['roofline']['achieved'], d['clocks'])"
