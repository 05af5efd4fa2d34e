mkdir -p gpurun_out
timeout 600 python scripts/tc_accuracy.py > gpurun_out/tc_acc2.log 2>&1; echo "acc rc=$?"; tail -20 gpurun_out/tc_acc2.log
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "all rc=$?"
tail -8 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_tc2.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/bench_tc2.log
