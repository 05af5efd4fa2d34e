# Two-chunk short-K tiles from TMEM (128-column tiles, kDirect 3) vs the
# promotion-register path (QSG_TC_DIRECT2=0): correctness, accuracy, speed.
mkdir -p gpurun_out/d2
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -m gpu -q -x -p no:cacheprovider > gpurun_out/d2/pytest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/d2/pytest.log
for v in QSG_TC_DIRECT2=1 QSG_TC_DIRECT2=0; do
  env $v timeout 900 python -m pytest tests/test_gpu_large.py -m gpu -q -p no:cacheprovider -k "config2 or config3s" > gpurun_out/d2/large_$v.log 2>&1; echo "$v large rc=$?"
  for c in config2 config3s; do echo "  $c $(python -c "
import json
d=json.load(open('gpurun_out/parity_$c.json')); print({k: (round(x['rel_l2'],8), round(x['max_rel_abs'],6)) for k, x in d.items() if 'vs' not in k and 'simt' not in k})")"; done
done
for r in 1 2; do
  for v in QSG_TC_DIRECT2=1 QSG_TC_DIRECT2=0; do
    for c in 4 3 2; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/d2/bench_c${c}_${v}_$r.log 2>&1
      echo "$v run $r c$c: $(tail -1 gpurun_out/d2/bench_c${c}_${v}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")')"
    done
  done
done
