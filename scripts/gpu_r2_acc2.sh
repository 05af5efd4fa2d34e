# Defaults now: 2 promotion chunks on k <= 256 tiles, accuracy split-K on the
# FP32 path for k >= 8192.  Full-size parity + kernel tests, SIMT speed, then
# the Bristlecone-70 reference fixture on the host.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -rA > gpurun_out/acc2_pytest.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED|SKIPPED" gpurun_out/acc2_pytest.log | tail -6
for c in config2 config5 config3s bc60; do echo "$c: $(python -c "
import json
d=json.load(open('gpurun_out/parity_$c.json')); print({k: (round(x['rel_l2'],8), round(x['max_rel_abs'],6)) for k, x in d.items() if 'vs' not in k})")"; done
timeout 600 python bench.py --config 2 --steps 2 --warmup 1 --no-tc --no-cpu-baseline > gpurun_out/acc2_simt_c2.log 2>&1; echo "simt c2: $(tail -1 gpurun_out/acc2_simt_c2.log | cut -c1-160)"
bash scripts/gpu_r2_golden2.sh
