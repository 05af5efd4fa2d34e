# Single-chunk tiles through the promotion path (QSG_TC_DIRECT=0: TMEM released right after one burst of loads, lane stores from registers) vs direct-from-TMEM: env A/B on configs 4, 3.
mkdir -p gpurun_out/dab
for r in 1 2; do
  for v in QSG_TC_DIRECT=1 QSG_TC_DIRECT=0; do
    for c in 4 3; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/dab/ops_c${c}_${v}_$r.jsonl > gpurun_out/dab/bench_c${c}_${v}_$r.log 2>&1
      echo "$v run $r c$c: $(tail -1 gpurun_out/dab/bench_c${c}_${v}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")') $(python scripts/prof_classes.py gpurun_out/dab/ops_c${c}_${v}_$r.jsonl | grep -E 'k=16     n=16 |k=128 ' | head -2 | tr -s ' ' | tr '\n' '|')"
    done
  done
done
