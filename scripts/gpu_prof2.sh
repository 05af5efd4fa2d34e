mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv $CMD > gpurun_out/ncu_launch2.log 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cgemm_tc2 -s 15 -c 1 -o gpurun_out/prof_tc2 $CMD > gpurun_out/ncu_tc2.log 2>&1; echo "ncu tc2 rc=$?"
timeout 900 python -m pytest tests/test_gpu_engine.py -m gpu -q -p no:cacheprovider -k full_size > gpurun_out/pytest_full.log 2>&1; echo "full rc=$?"; tail -3 gpurun_out/pytest_full.log
