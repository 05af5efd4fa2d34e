# A/B: raw-A stage conversion serviced between epilogue slabs (default) vs
# converted ahead of the previous chunk's epilogue (QSG_TC_SERVICE=0).
mkdir -p gpurun_out
for r in 1 2; do
  for v in QSG_TC_SERVICE=1 QSG_TC_SERVICE=0; do
    for c in 4 2; do
      env $v python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --profile-out gpurun_out/abs_c${c}_${v}_$r.jsonl > gpurun_out/abs_c${c}_${v}_$r.log 2>&1
      echo "$v run $r c$c: $(tail -1 gpurun_out/abs_c${c}_${v}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],1), "ms/step", d["clocks"]["sm_mhz"], "MHz")')"
    done
  done
done
python scripts/prof_classes.py gpurun_out/abs_c4_QSG_TC_SERVICE=1_2.jsonl gpurun_out/abs_c4_QSG_TC_SERVICE=0_2.jsonl
