# Lane-per-row STG.256 split stores (QSG_TC_LANESTORE): correctness, then A/B on configs 4, 3, 2, 5.
mkdir -p gpurun_out/ls
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_large.py tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ls/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ls/pytest.log
for r in 1 2; do
  for v in QSG_TC_LANESTORE=1 QSG_TC_LANESTORE=0; do
    for c in 4 3 2 5; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/ls/ops_c${c}_${v}_$r.jsonl > gpurun_out/ls/bench_c${c}_${v}_$r.log 2>&1
      echo "$v run $r c$c: $(tail -1 gpurun_out/ls/bench_c${c}_${v}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")') $(python scripts/prof_classes.py gpurun_out/ls/ops_c${c}_${v}_$r.jsonl | sed -n 2,3p | tr -s ' ' | tr '\n' '|')"
    done
  done
done
