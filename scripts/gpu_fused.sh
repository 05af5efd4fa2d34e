mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "all rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fused.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_fused.log').read().strip().splitlines()[-1]);print(d['value'], d['tflops_eq1'], d['roofline']['achieved'], d['roofline']['permute_share_of_step'], d['clocks'])"
timeout 900 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c4_fused.log 2>&1; echo "c4 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_c4_fused.log').read().strip().splitlines()[-1]);print(d['value'], d['tflops_eq1'], d['roofline']['permute_share_of_step'], d['clocks'])"
timeout 900 python bench.py --config 5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c5_fused.log 2>&1; echo "c5 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_c5_fused.log').read().strip().splitlines()[-1]);print(d['value'], d['tflops_eq1'], d['roofline']['permute_share_of_step'], d['clocks'])"
