# Round-2 check: GPU tests, smoke, default bench (config 5) with the CPU
# baseline, and config 2 without it.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_pytest.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_smoke.log
timeout 900 python bench.py --steps 6 --warmup 3 > gpurun_out/r2_bench_c5.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2_bench_c5.log | cut -c1-600
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c2.log 2>&1; echo "c2 rc=$?"; tail -1 gpurun_out/r2_bench_c2.log | cut -c1-400
