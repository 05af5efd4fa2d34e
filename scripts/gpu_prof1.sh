mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r1.log
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cgemm_tc_kernel -s 9 -c 1 -o gpurun_out/prof_tc $CMD > gpurun_out/ncu_tc.log 2>&1; echo "ncu tc rc=$?"
ncu --set full --clock-control none --import-source on -k regex:permute_bits -s 40 -c 1 -o gpurun_out/prof_perm $CMD > gpurun_out/ncu_perm.log 2>&1; echo "ncu perm rc=$?"
ls -la gpurun_out
