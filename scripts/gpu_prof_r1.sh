# Round-1 evidence: launch list of the default bench command + ncu --set full of the
# dominant launch (s026) and of one n=256 step (s013), current code.
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/plain_r1.log 2>&1 || { echo "plain failed"; tail gpurun_out/plain_r1.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_launch_r1.log 2>&1; echo "ncu list rc=$?"
IDX=$(python scripts/ncu_pick.py gpurun_out/launches_r1.csv cgemm_f16_pair_kernel --summary 2> gpurun_out/launches_r1_summary.txt); echo "idx=$IDX"; head -12 gpurun_out/launches_r1_summary.txt
ncu --set full --clock-control none --import-source on -k regex:cgemm_f16_pair -s $IDX -c 1 -o gpurun_out/prof_r1_s026 $CMD > gpurun_out/ncu_r1_s026.log 2>&1; echo "ncu s026 rc=$?"
IDX2=$(python scripts/ncu_pick.py gpurun_out/launches_r1.csv cgemm_f16_pair_kernel --ms=10 --ms=16); echo "idx2=$IDX2"
ncu --set full --clock-control none --import-source on -k regex:cgemm_f16_pair -s $IDX2 -c 1 -o gpurun_out/prof_r1_s013 $CMD > gpurun_out/ncu_r1_s013.log 2>&1; echo "ncu s013 rc=$?"
