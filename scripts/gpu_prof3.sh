mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/plain6.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches6.csv $CMD > gpurun_out/ncu_launch6.log 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:cgemm_tc2 -s 20 -c 1 -o gpurun_out/prof_s026_v3 $CMD > gpurun_out/ncu_s026_v3.log 2>&1; echo "ncu s026 rc=$?"
