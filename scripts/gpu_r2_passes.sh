# Power model: 3 vs 2 MMA passes per K16 step (2 is numerically wrong; it
# only measures how throughput at the power cap scales with the MMA count).
mkdir -p gpurun_out
for r in 1 2; do
  for v in QSG_TC_PASSES=3 QSG_TC_PASSES=2; do
    for c in 5 2; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/pp_c${c}_${v}_$r.log 2>&1
      echo "$v run $r c$c: $(tail -1 gpurun_out/pp_c${c}_${v}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],1), "ms/step", d["clocks"]["sm_mhz"], "MHz", d["clocks"]["reasons"])')"
    done
  done
done
