# ncu --set full of the first cgemm_f16_pair launch whose duration is in [LO, HI] ms (config CFG).
mkdir -p gpurun_out
CMD="python bench.py --config ${CFG:-2} --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/plain_win.log 2>&1 || { echo "plain failed"; tail gpurun_out/plain_win.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_win.csv $CMD > gpurun_out/ncu_launch_win.log 2>&1; echo "ncu list rc=$?"
IDX=$(python scripts/ncu_pick.py gpurun_out/launches_win.csv cgemm_f16_pair_kernel --ms=$LO --ms=$HI --summary 2> gpurun_out/launches_win_summary.txt); echo "idx=$IDX"; head -5 gpurun_out/launches_win_summary.txt
ncu --set full --clock-control none --import-source on -k regex:cgemm_f16_pair -s $IDX -c 1 -o gpurun_out/prof_${TAG:-win} $CMD > gpurun_out/ncu_win.log 2>&1; echo "ncu rc=$?"
