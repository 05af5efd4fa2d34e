# Correctness of the early-release kDirect variant, then A/B vs slab-by-slab TMEM reads.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ae_pytest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ae_pytest.log
for r in 1 2; do
  for v in QSG_TC_EARLY=1 QSG_TC_EARLY=0; do
    for c in 4 3 2; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/ae_c${c}_${v}_$r.jsonl > gpurun_out/ae_c${c}_${v}_$r.log 2>&1
      echo "$v run $r c$c: $(tail -1 gpurun_out/ae_c${c}_${v}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")')"
    done
  done
done
python scripts/prof_classes.py gpurun_out/ae_c4_QSG_TC_EARLY=1_2.jsonl gpurun_out/ae_c4_QSG_TC_EARLY=0_2.jsonl
