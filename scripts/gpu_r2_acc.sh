# Accuracy knobs on config 2 at full size vs fp64 (test_gpu_large writes
# gpurun_out/parity_config2.json): default, promotion every 128 real K on
# every GEMM (QSG_TC_CHUNK=4), and the 2x2 embedding on the big steps (QSG_TC_3M=0).
mkdir -p gpurun_out/acc
for v in BASE=1 QSG_TC_CHUNK=4 QSG_TC_3M=0; do
  env $v timeout 900 python -m pytest tests/test_gpu_large.py -m gpu -q -p no:cacheprovider -k config2 > gpurun_out/acc/$v.log 2>&1
  cp gpurun_out/parity_config2.json gpurun_out/acc/parity_config2_$v.json
  echo "$v: $(python -c "import json; d=json.load(open('gpurun_out/acc/parity_config2_$v.json')); print({k: (round(v['rel_l2'],8), round(v['max_rel_abs'],6)) for k, v in d.items()})")"
done
