# 3M complex products: kernel tests, full-size parity (configs 2 / 5 run the
# 3M path on their big steps), then A/B against the 2x2 embedding.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider > gpurun_out/m3_kernels.log 2>&1; echo "kernel tests rc=$?"; tail -3 gpurun_out/m3_kernels.log
timeout 900 python -m pytest tests/test_gpu_large.py -m gpu -q -p no:cacheprovider -k "config5 or config2" > gpurun_out/m3_large.log 2>&1; echo "large rc=$?"; tail -3 gpurun_out/m3_large.log
cat gpurun_out/parity_config2.json gpurun_out/parity_config5.json | python -c "import sys; print(sys.stdin.read()[:3000])"
for r in 1 2; do
  for v in QSG_TC_3M=1 QSG_TC_3M=0; do
    for c in 5 2; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/m3_c${c}_${v}_$r.jsonl > gpurun_out/m3_c${c}_${v}_$r.log 2>&1
      echo "$v run $r c$c: $(tail -1 gpurun_out/m3_c${c}_${v}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],1), "ms/step", d["clocks"]["sm_mhz"], "MHz", round(d["tflops_eq1"],1), "TF/s")')"
    done
  done
done
python scripts/prof_classes.py gpurun_out/m3_c5_QSG_TC_3M=1_2.jsonl gpurun_out/m3_c2_QSG_TC_3M=1_2.jsonl
