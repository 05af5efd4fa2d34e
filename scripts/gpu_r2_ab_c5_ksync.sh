# Config 5 same-box check of the K-sync change (previous build vs HEAD).
mkdir -p gpurun_out/c5ab
for r in 1 2; do
  for v in "QSG_LIB=$PWD/ab/libqsg_base.so" "QSG_LIB=$PWD/paper_1905_00444_b200/libqsg.so"; do
    tag=$(basename ${v#QSG_LIB=} .so)
    env $v python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c5ab/bench_${tag}_$r.log 2>&1
    echo "$tag run $r c5: $(tail -1 gpurun_out/c5ab/bench_${tag}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")')"
  done
done
