# Two-step lookahead output layouts (QSG_LAYOUT2): correctness, then A/B on configs 4, 3, 2, 5.
mkdir -p gpurun_out/l2
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_large.py -m gpu -q -x -p no:cacheprovider > gpurun_out/l2/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/l2/pytest.log
for r in 1 2; do
  for v in QSG_LAYOUT2=1 QSG_LAYOUT2=0; do
    for c in 4 3 2 5; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/l2/ops_c${c}_${v}_$r.jsonl > gpurun_out/l2/bench_c${c}_${v}_$r.log 2>&1
      echo "$v run $r c$c: $(tail -1 gpurun_out/l2/bench_c${c}_${v}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")') $(python scripts/prof_classes.py gpurun_out/l2/ops_c${c}_${v}_$r.jsonl | sed -n 2p | tr -s ' ')"
    done
  done
done
