# FP32 streaming kernel for the n = k = 16 split-in / split-out bond-closing steps (QSG_TC_NARROW):
# GPU tests (full-size Bristlecone parity included), then env A/B on configs 4, 3.
# (Record of the A/B in profiles/r2/narrow_fp32/: the kernel was removed afterwards, so QSG_TC_NARROW is no longer read.)
mkdir -p gpurun_out/abnw
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_large.py -m gpu -q -x -p no:cacheprovider > gpurun_out/abnw/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/abnw/pytest.log
cp gpurun_out/parity_*.json gpurun_out/abnw/ 2>/dev/null
for r in 1 2; do
  for v in QSG_TC_NARROW=1 QSG_TC_NARROW=0; do
    for c in 4 3; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/abnw/ops_c${c}_${v}_$r.jsonl > gpurun_out/abnw/bench_c${c}_${v}_$r.log 2>&1
      echo "$v run $r c$c: $(tail -1 gpurun_out/abnw/bench_c${c}_${v}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")') $(python scripts/prof_classes.py gpurun_out/abnw/ops_c${c}_${v}_$r.jsonl | grep -E 'k=16     n=16 ' | head -2 | tr -s ' ' | tr '\n' '|')"
    done
  done
done
