mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "tensor_core" -p no:cacheprovider -x > gpurun_out/pytest_tc.log 2>&1; echo "tc rc=$?"
tail -30 gpurun_out/pytest_tc.log
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "all rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_tc.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/bench_tc.log
