mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py -m gpu -q -x -p no:cacheprovider -k "widened or config1" > gpurun_out/c1_pytest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/c1_pytest.log
for r in 1 2; do
timeout 600 python bench.py --config 1 --steps 50 --warmup 5 > gpurun_out/c1_bench_$r.log 2>&1; echo "c1 rc=$?"; tail -1 gpurun_out/c1_bench_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["ms_per_step"], d["roofline"]["kernel"], d["roofline"]["achieved"], d["roofline"]["frac"], d["cpu_baseline"]["value"])'
done
