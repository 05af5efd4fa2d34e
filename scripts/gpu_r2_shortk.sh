# Short-K (k <= 256) promotion chunks: accuracy (config 2 / 6x10 stand-in vs
# fp64 + reference) and speed (configs 2, 3, 4).
mkdir -p gpurun_out/sk
for v in QSG_TC_SHORTK_CHUNKS=1 QSG_TC_SHORTK_CHUNKS=2 QSG_TC_SHORTK_CHUNKS=4; do
  env $v timeout 900 python -m pytest tests/test_gpu_large.py -m gpu -q -p no:cacheprovider -k "config2 or config3s" > gpurun_out/sk/$v.log 2>&1
  for c in config2 config3s; do cp gpurun_out/parity_$c.json gpurun_out/sk/parity_${c}_$v.json; done
  echo "$v accuracy: $(python -c "
import json
for c in ('config2','config3s'):
    d=json.load(open('gpurun_out/sk/parity_%s_$v.json' % c)); print(c, {k: (round(x['rel_l2'],8), round(x['max_rel_abs'],6)) for k, x in d.items() if 'vs' not in k})")"
  for c in 2 4 3; do
    env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/sk/bench_c${c}_$v.log 2>&1
    echo "$v c$c: $(tail -1 gpurun_out/sk/bench_c${c}_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")')"
  done
done
