# Config 4: ncu --set full of the m = 2^27, n = k = 16 bond-closing launch
# (cgemm_f16_pair_kernel<32, ...>, the longest launch of that variant).
mkdir -p gpurun_out
CMD="python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pn_launches.csv $CMD > gpurun_out/pn_ncu_list.log 2>&1; echo "ncu list rc=$?"
IDX=$(python scripts/ncu_pick.py gpurun_out/pn_launches.csv cgemm_f16_pair_kernel "--variant=cgemm_f16_pair_kernel<32, 1, 64, 1"); echo "idx=$IDX"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cgemm_f16_pair_kernel -s $IDX -c 1 -o gpurun_out/prof_c4_narrow $CMD > gpurun_out/pn_ncu_full.log 2>&1; echo "ncu rc=$?"
