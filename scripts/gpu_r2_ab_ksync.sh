# K-sync off for single-column-tile launches (no shared A slabs): tests, same-box A/B on configs 4, 3, 2.
mkdir -p gpurun_out/abk
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_large.py -m gpu -q -x -p no:cacheprovider > gpurun_out/abk/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/abk/pytest.log
for r in 1 2; do
  for v in "QSG_LIB=$PWD/ab/libqsg_base.so" "QSG_LIB=$PWD/paper_1905_00444_b200/libqsg.so"; do
    tag=$(basename ${v#QSG_LIB=} .so)
    for c in 4 3 2; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/abk/ops_c${c}_${tag}_$r.jsonl > gpurun_out/abk/bench_c${c}_${tag}_$r.log 2>&1
      echo "$tag run $r c$c: $(tail -1 gpurun_out/abk/bench_c${c}_${tag}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")') $(python scripts/prof_classes.py gpurun_out/abk/ops_c${c}_${tag}_$r.jsonl | grep -E 'k=16 ' | head -2 | tr -s ' ' | tr '\n' '|')"
    done
  done
done
