# Config 5 under rasterisation group sizes (QSG_TC_GROUPM): DRAM re-reads of the cubes vs power-capped clocks.
mkdir -p gpurun_out/gm
for r in 1 2; do
  for v in QSG_TC_GROUPM=8 QSG_TC_GROUPM=4 QSG_TC_GROUPM=16 QSG_TC_GROUPM=9; do
    env $v python bench.py --config 5 --steps 4 --warmup 2 --no-cpu-baseline > gpurun_out/gm/bench_${v}_$r.log 2>&1
    echo "$v run $r: $(tail -1 gpurun_out/gm/bench_${v}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")')"
  done
done
