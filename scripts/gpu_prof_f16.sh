mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/plain_f16c.log 2>&1 || { echo "plain failed"; tail gpurun_out/plain_f16.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_f16c.csv $CMD > gpurun_out/ncu_launch_f16c.log 2>&1; echo "ncu list rc=$?"
IDX=$(python scripts/ncu_pick.py gpurun_out/launches_f16c.csv cgemm_f16_pair_kernel --summary 2> gpurun_out/launches_f16c_summary.txt); echo "idx=$IDX"; cat gpurun_out/launches_f16c_summary.txt
ncu --set full --clock-control none --import-source on -k regex:cgemm_f16_pair -s $IDX -c 1 -o gpurun_out/prof_s026_f16c $CMD > gpurun_out/ncu_s026_f16c.log 2>&1; echo "ncu s026 rc=$?"
