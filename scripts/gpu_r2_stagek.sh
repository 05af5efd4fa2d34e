# 32-K stages (6 in flight) for the short-K pre-split tiles (QSG_TC_STAGEK=32)
# vs 64-K stages: correctness then speed on configs 4, 3, 2.
mkdir -p gpurun_out/stk
QSG_TC_STAGEK=32 timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_large.py -m gpu -q -x -p no:cacheprovider -k "split or config2 or config3s or bc70" > gpurun_out/stk/pytest.log 2>&1; echo "tests(stagek32) rc=$?"; tail -2 gpurun_out/stk/pytest.log
for r in 1 2; do
  for v in QSG_TC_STAGEK=32 QSG_TC_STAGEK=64; do
    for c in 4 3 2; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/stk/ops_c${c}_${v}_$r.jsonl > gpurun_out/stk/bench_c${c}_${v}_$r.log 2>&1
      echo "$v run $r c$c: $(tail -1 gpurun_out/stk/bench_c${c}_${v}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")') $(python scripts/prof_classes.py gpurun_out/stk/ops_c${c}_${v}_$r.jsonl | sed -n 2p | tr -s ' ')"
    done
  done
done
# config 1: per-launch durations + DRAM bytes of one widened contraction (latency-floor evidence)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/stk/ncu_launches_c1.csv python bench.py --config 1 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/stk/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"
