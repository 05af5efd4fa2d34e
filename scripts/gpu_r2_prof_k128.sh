# Config 4: ncu --set full of the k = 128, n = 256 pair launch (step 93,
# m = 2^23; the only <256,1,64,0> launch of 9.0-9.5 ms under ncu; k = 256 launches at m = 2^23 take 8.2-8.5), two promotion chunks.
mkdir -p gpurun_out
CMD="python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pk128_launches.csv $CMD > gpurun_out/pk128_ncu_list.log 2>&1; echo "ncu list rc=$?"
IDX=$(python scripts/ncu_pick.py gpurun_out/pk128_launches.csv cgemm_f16_pair_kernel "--variant=cgemm_f16_pair_kernel<256, 1, 64, 0>" --ms=9.0 --ms=9.5); echo "idx=$IDX"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cgemm_f16_pair_kernel -s $IDX -c 1 -o gpurun_out/prof_c4_k128 $CMD > gpurun_out/pk128_ncu_full.log 2>&1; echo "ncu rc=$?"
