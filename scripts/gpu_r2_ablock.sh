# k-blocked A hand-offs (QSG_ABLOCK): correctness at full size, then A/B on configs 4, 3, 2, 5.
mkdir -p gpurun_out/ab
timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_large.py tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab/pytest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab/pytest.log
for c in config2 config3s bc70; do echo "$c $(python -c "
import json; d=json.load(open('gpurun_out/parity_$c.json')); print({k: (round(x['rel_l2'],8), round(x['max_rel_abs'],6)) for k, x in d.items() if 'vs' not in k and 'simt' not in k})")"; done
for r in 1 2; do
  for v in QSG_ABLOCK=1 QSG_ABLOCK=0; do
    for c in 4 3 2 5; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/ab/ops_c${c}_${v}_$r.jsonl > gpurun_out/ab/bench_c${c}_${v}_$r.log 2>&1
      echo "$v run $r c$c: $(tail -1 gpurun_out/ab/bench_c${c}_${v}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")') $(python scripts/prof_classes.py gpurun_out/ab/ops_c${c}_${v}_$r.jsonl | sed -n 2p | tr -s ' ')"
    done
  done
done
