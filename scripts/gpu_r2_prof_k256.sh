# TMEM ld microbenchmark + ncu of config 4 (Bristlecone-70)'s k=256 class:
# the launch list, then one --set full capture of the longest pair launch.
mkdir -p gpurun_out
./scripts/micro/tmem_ld_bw > gpurun_out/tmem_ld_bw.txt 2>&1; cat gpurun_out/tmem_ld_bw.txt
CMD="python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/c4p_plain.log 2>&1 || { echo "plain failed"; tail gpurun_out/c4p_plain.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4p_launches.csv $CMD > gpurun_out/c4p_ncu_list.log 2>&1; echo "ncu list rc=$?"
IDX=$(python scripts/ncu_pick.py gpurun_out/c4p_launches.csv cgemm_f16_pair_kernel --summary 2> gpurun_out/c4p_launches_summary.txt); echo "idx=$IDX"; head -12 gpurun_out/c4p_launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cgemm_f16_pair -s $IDX -c 1 -o gpurun_out/prof_c4k256 $CMD > gpurun_out/c4p_ncu_full.log 2>&1; echo "ncu rc=$?"
