mkdir -p gpurun_out/c2k
timeout 900 python -m pytest tests/test_gpu_engine.py -m gpu -q -p no:cacheprovider -rA -k "failure or run_amplitudes or widened" > gpurun_out/c2k/pytest.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/c2k/pytest.log | tail -4
timeout 300 python bench.py --config 1 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c2k/c1_s1.log 2>&1; echo "c1 steps=1 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c2k/ncu_launches_c1.csv python bench.py --config 1 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/c2k/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"
