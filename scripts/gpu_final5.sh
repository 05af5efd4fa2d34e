# Final evidence for the committed code: GPU suite, smoke, default bench
# (+CPU baseline), reference arm, config 1 (+CPU baseline), launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/f5_pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/f5_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f5_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f5_smoke.log
timeout 900 python bench.py > gpurun_out/f5_bench_c2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/f5_bench_c2.log | cut -c1-160
timeout 900 python bench.py --impl reference > gpurun_out/f5_ref_c2.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/f5_ref_c2.log | cut -c1-160
timeout 900 python bench.py --config 1 > gpurun_out/f5_bench_c1.log 2>&1; echo "c1 rc=$?"; tail -1 gpurun_out/f5_bench_c1.log | cut -c1-160
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f5_launches.csv $CMD > gpurun_out/f5_ncu_list.log 2>&1; echo "ncu list rc=$?"
python scripts/ncu_pick.py gpurun_out/f5_launches.csv cgemm_f16_pair_kernel --summary 2> gpurun_out/f5_launches_summary.txt; head -8 gpurun_out/f5_launches_summary.txt
