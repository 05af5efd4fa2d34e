# Final state: GPU suite, smoke, default bench (+CPU baseline), configs 1/3/4/5, accuracy study.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/f4_pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/f4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f4_smoke.log
timeout 900 python bench.py > gpurun_out/f4_bench_c2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/f4_bench_c2.log | cut -c1-160
for c in 1 3 4 5; do
  timeout 900 python bench.py --config $c > gpurun_out/f4_bench_c$c.log 2>&1; echo "c$c rc=$?"; tail -1 gpurun_out/f4_bench_c$c.log | cut -c1-120
done
timeout 600 python scripts/tc_accuracy.py > gpurun_out/f4_acc.log 2>&1; tail -1 gpurun_out/f4_acc.log
