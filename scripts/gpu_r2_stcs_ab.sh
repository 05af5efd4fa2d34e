# Evict-first output stores (QSG_TC_STCS, default on) re-checked with the lane-store epilogue: env A/B on configs 4, 2, 5.
mkdir -p gpurun_out/stcs
for r in 1 2; do
  for v in QSG_TC_STCS=1 QSG_TC_STCS=0; do
    for c in 4 2 5; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/stcs/bench_c${c}_${v}_$r.log 2>&1
      echo "$v run $r c$c: $(tail -1 gpurun_out/stcs/bench_c${c}_${v}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")')"
    done
  done
done
