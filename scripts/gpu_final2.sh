# Round-end evidence with the final code: GPU tests, smoke, the default bench
# line (with the CPU baseline), the reference arm, configs 1/3/4/5, the launch
# list of the default bench and ncu --set full of its dominant launch.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/f2_pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/f2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f2_smoke.log
timeout 900 python bench.py > gpurun_out/f2_bench_c2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/f2_bench_c2.log | cut -c1-160
timeout 900 python bench.py --impl reference > gpurun_out/f2_ref_c2.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/f2_ref_c2.log | cut -c1-160
for c in 1 3 4 5; do
  timeout 900 python bench.py --config $c > gpurun_out/f2_bench_c$c.log 2>&1; echo "c$c rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/f2_bench_c$c.log').read().strip().splitlines()[-1]);print('   ', d['value'], round(d['tflops_eq1'],1), round(d['roofline']['achieved'],1), round(d['roofline']['frac'],3), d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d.get('cpu_baseline',{}).get('value'))"
done
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f2_launches.csv $CMD > gpurun_out/f2_ncu_list.log 2>&1; echo "ncu list rc=$?"
IDX=$(python scripts/ncu_pick.py gpurun_out/f2_launches.csv cgemm_f16_pair_kernel --summary 2> gpurun_out/f2_launches_summary.txt); echo "idx=$IDX"; head -8 gpurun_out/f2_launches_summary.txt
ncu --set full --clock-control none --import-source on -k regex:cgemm_f16_pair -s $IDX -c 1 -o gpurun_out/f2_s026 $CMD > gpurun_out/f2_ncu_full.log 2>&1; echo "ncu full rc=$?"
