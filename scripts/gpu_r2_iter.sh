# Iteration check: GPU tests, then bench lines for configs 4, 3, 2, 5 with per-op profiles.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/it_pytest.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/it_pytest.log
for c in 4 3 2 5; do
  timeout 900 python bench.py --config $c --steps 4 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/it_ops_c$c.jsonl > gpurun_out/it_bench_c$c.log 2>&1; echo "c$c rc=$?"; tail -1 gpurun_out/it_bench_c$c.log | cut -c1-250
done
