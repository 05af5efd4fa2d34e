# Full GPU suite + headline bench lines, with the reference anchor (one
# complete stock reference slice, 1 thread) running on the host meanwhile.
mkdir -p gpurun_out
(OPENBLAS_NUM_THREADS=1 timeout 2400 python scripts/ref_anchor.py --out gpurun_out/ref_anchor.json > gpurun_out/ref_anchor.log 2>&1 &)
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rA > gpurun_out/full_pytest.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED|SKIPPED" gpurun_out/full_pytest.log | tail -8
for c in 5 2; do
  timeout 900 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --profile-out gpurun_out/full_ops_c$c.jsonl > gpurun_out/full_bench_c$c.log 2>&1; echo "c$c rc=$?"; tail -1 gpurun_out/full_bench_c$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], round(d["ms_per_step"],1), "ms/step", d["clocks"]["sm_mhz"], "MHz", round(d["tflops_eq1"],1), "TF/s", d["roofline"]["kernel"], round(d["roofline"]["frac"],3))'
done
# wait for the anchor (bounded)
for i in $(seq 1 60); do [ -s gpurun_out/ref_anchor.json ] && break; sleep 20; done
cat gpurun_out/ref_anchor.json; tail -3 gpurun_out/ref_anchor.log
