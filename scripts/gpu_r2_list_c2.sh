mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python bench.py --config 2 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/c2_ncu_list.log 2>&1; echo "ncu list rc=$?"
python scripts/ncu_pick.py gpurun_out/c2_launches.csv cgemm_f16_pair_kernel --summary 2>&1 | head -20
