# k <= 128 tiles as one 256-real-K chunk (same chunk length as k = 256 tiles):
# GPU tests (incl. full-size parity: Bristlecone-70 has k = 128 steps), same-box
# A/B against the previous build on configs 4, 3, 2, then ncu --set full of
# config 4's k = n = 256 lane-store launch (m = 2^23).
mkdir -p gpurun_out/abc
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_large.py -m gpu -q -x -p no:cacheprovider > gpurun_out/abc/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/abc/pytest.log
cp gpurun_out/parity_*.json gpurun_out/abc/ 2>/dev/null
for r in 1 2; do
  for v in "QSG_LIB=$PWD/ab/libqsg_base.so" "QSG_LIB=$PWD/paper_1905_00444_b200/libqsg.so"; do
    tag=$(basename ${v#QSG_LIB=} .so)
    for c in 4 3 2; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/abc/ops_c${c}_${tag}_$r.jsonl > gpurun_out/abc/bench_c${c}_${tag}_$r.log 2>&1
      echo "$tag run $r c$c: $(tail -1 gpurun_out/abc/bench_c${c}_${tag}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")') $(python scripts/prof_classes.py gpurun_out/abc/ops_c${c}_${tag}_$r.jsonl | grep -E 'k=128 |k=64 ' | tr -s ' ' | tr '\n' '|')"
    done
  done
done
C4="python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/abc/ncu_launches_c4.csv $C4 > /dev/null 2>&1; echo "ncu list rc=$?"
IDX4=$(python scripts/ncu_pick.py gpurun_out/abc/ncu_launches_c4.csv cgemm_f16_pair_kernel "--variant=cgemm_f16_pair_kernel<256, 1, 64, 0, 1>" --ms=7.0 --ms=9.0 --skip=1); echo "idx4=$IDX4"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cgemm_f16_pair_kernel -s $IDX4 -c 1 -o gpurun_out/abc/ncu_full_c4_k256 $C4 > gpurun_out/abc/ncu_full_c4.log 2>&1; echo "ncu c4 rc=$?"
