# SIMT split-K for few-tile GEMMs with 32 <= k < 512: GPU tests, then same-box A/B vs the previous build.
mkdir -p gpurun_out/abs
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/abs/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/abs/pytest.log
cp gpurun_out/parity_*.json gpurun_out/abs/ 2>/dev/null
for r in 1 2; do
  for v in "QSG_LIB=$PWD/ab/libqsg_base.so" "QSG_LIB=$PWD/paper_1905_00444_b200/libqsg.so"; do
    tag=$(basename ${v#QSG_LIB=} .so)
    for c in 3 4 2; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/abs/ops_c${c}_${tag}_$r.jsonl > gpurun_out/abs/bench_c${c}_${tag}_$r.log 2>&1
      echo "$tag run $r c$c: $(tail -1 gpurun_out/abs/bench_c${c}_${tag}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")') $(python scripts/prof_classes.py gpurun_out/abs/ops_c${c}_${tag}_$r.jsonl | grep -E 'total' | tr -s ' ' | tr '\n' '|')"
    done
  done
done
