# Config 4 (Bristlecone-70, clustered plan): launch list, then ncu --set full
# of the longest k = n = 256 pair launch (split-in / split-out, kDirect).
mkdir -p gpurun_out
CMD="python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pc4_launches.csv $CMD > gpurun_out/pc4_ncu_list.log 2>&1; echo "ncu list rc=$?"
IDX=$(python scripts/ncu_pick.py gpurun_out/pc4_launches.csv cgemm_f16_pair_kernel "--variant=cgemm_f16_pair_kernel<256, 1, 64, 1>" --summary 2> gpurun_out/pc4_launches_summary.txt); echo "idx=$IDX"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cgemm_f16_pair_kernel -s $IDX -c 1 -o gpurun_out/prof_c4_split256 $CMD > gpurun_out/pc4_ncu_full.log 2>&1; echo "ncu rc=$?"
