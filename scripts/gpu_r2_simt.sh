# FP32-FFMA kernel: 16-byte B loads / C stores (column pairs): correctness + speed (--no-tc).
mkdir -p gpurun_out/simt
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -m gpu -q -x -p no:cacheprovider > gpurun_out/simt/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/simt/pytest.log
timeout 900 python -m pytest tests/test_gpu_large.py -m gpu -q -p no:cacheprovider -k "config2" > gpurun_out/simt/large.log 2>&1; echo "large rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/parity_config2.json')); print({k: (round(x['rel_l2'],8), round(x['max_rel_abs'],6)) for k, x in d.items() if 'vs' not in k})"
for c in 2 5; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 1 --no-tc --no-cpu-baseline > gpurun_out/simt/bench_c$c.log 2>&1
  echo "c$c --no-tc: $(tail -1 gpurun_out/simt/bench_c$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["value"], round(d["ms_per_step"],1), "ms", d["clocks"]["sm_mhz"], "MHz", r["kernel"], round(r["achieved"],1), round(r["frac"],3))')"
done
