# ncu --set full of config 3's first k=256 n=256 launch (step 6, ~1.3 ms) with the current code.
mkdir -p gpurun_out
CMD="python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/c3b_plain.log 2>&1 || { echo "plain failed"; tail gpurun_out/c3b_plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3b_launches.csv $CMD > gpurun_out/c3b_ncu_list.log 2>&1; echo "ncu list rc=$?"
IDX=$(python scripts/ncu_pick.py gpurun_out/c3b_launches.csv cgemm_f16_pair_kernel --ms=1.15 --ms=2.0 --summary 2> gpurun_out/c3b_launches_summary.txt); echo "idx=$IDX"; head -8 gpurun_out/c3b_launches_summary.txt
ncu --set full --clock-control none --import-source on -k regex:cgemm_f16_pair -s $IDX -c 1 -o gpurun_out/prof_c3k256 $CMD > gpurun_out/c3b_ncu_full.log 2>&1; echo "ncu rc=$?"
