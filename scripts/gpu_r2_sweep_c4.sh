# Config 4 (Bristlecone-70) knob sweep on the current build (narrow tiles now
# keep up to 8 TMEM buffers): K-sync spacing, rasterisation group, streaming
# stores.  Per-op class totals from the profiling pass.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -m gpu -q -x -p no:cacheprovider > gpurun_out/sw_pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/sw_pytest.log
for v in BASE=1 QSG_TC_SYNC=0 QSG_TC_SYNC=4 QSG_TC_SYNC=64 QSG_TC_GROUPM=2 QSG_TC_GROUPM=32 QSG_TC_STCS=0; do
  env $v python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/sw_c4_$v.jsonl > gpurun_out/sw_c4_$v.log 2>&1
  echo "$v: $(tail -1 gpurun_out/sw_c4_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")') $(python scripts/prof_classes.py gpurun_out/sw_c4_$v.jsonl | sed -n 2,3p | tr -s ' ' | tr '\n' '|')"
done
