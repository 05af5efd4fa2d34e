# Round-end evidence with the current code: GPU tests, smoke, default bench line,
# the launch list of the bench command and ncu --set full of its dominant launch.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/final_bench.log | cut -c1-200
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv $CMD > gpurun_out/final_ncu_list.log 2>&1; echo "ncu list rc=$?"
IDX=$(python scripts/ncu_pick.py gpurun_out/final_launches.csv cgemm_f16_pair_kernel --summary 2> gpurun_out/final_launches_summary.txt); echo "idx=$IDX"; head -8 gpurun_out/final_launches_summary.txt
ncu --set full --clock-control none --import-source on -k regex:cgemm_f16_pair -s $IDX -c 1 -o gpurun_out/final_s026 $CMD > gpurun_out/final_ncu_full.log 2>&1; echo "ncu full rc=$?"
