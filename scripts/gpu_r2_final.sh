# Round-end evidence: GPU tests, smoke, the default bench line exactly as the
# driver runs it (config 5, 20 steps, CPU baseline), the reference arm, the
# other configs' lines, and the ncu launch list + one --set full capture of
# the dominant kernel (config 5: a 3M product launch of a 2^15 cube).
mkdir -p gpurun_out/final
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rA > gpurun_out/final/pytest_gpu.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|FAILED|SKIPPED" gpurun_out/final/pytest_gpu.log | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final/smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final/bench_c5.jsonl 2> gpurun_out/final/bench_c5.err; echo "bench rc=$?"; tail -1 gpurun_out/final/bench_c5.jsonl | cut -c1-300
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/final/bench_ref_c5.jsonl 2> gpurun_out/final/bench_ref_c5.err; echo "ref rc=$?"; tail -1 gpurun_out/final/bench_ref_c5.jsonl | cut -c1-300
for c in 2 4 3 1; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --profile-out gpurun_out/final/ops_c$c.jsonl > gpurun_out/final/bench_c$c.jsonl 2> gpurun_out/final/bench_c$c.err; echo "c$c rc=$?"; tail -1 gpurun_out/final/bench_c$c.jsonl | cut -c1-200
done
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/ncu_launches_c5.csv $CMD > gpurun_out/final/ncu_list.log 2>&1; echo "ncu list rc=$?"
IDX=$(python scripts/ncu_pick.py gpurun_out/final/ncu_launches_c5.csv cgemm_f16_pair_kernel --summary 2> gpurun_out/final/ncu_launches_c5_summary.txt); echo "idx=$IDX"; head -8 gpurun_out/final/ncu_launches_c5_summary.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cgemm_f16_pair_kernel -s $IDX -c 1 -o gpurun_out/final/ncu_full_c5_cube $CMD > gpurun_out/final/ncu_full.log 2>&1; echo "ncu rc=$?"
# config 1: per-launch durations of one widened contraction (latency floor evidence)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final/ncu_launches_c1.csv python bench.py --config 1 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/final/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"
# config 4 (Bristlecone-70): --set full of its dominant class, the k = n = 256 lane-store launch
# (m = 2^23; --skip=1 passes over the first 7-9 ms launch of the variant, the n = 2048 step)
C4="python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/ncu_launches_c4.csv $C4 > gpurun_out/final/ncu_list_c4.log 2>&1; echo "ncu list c4 rc=$?"
IDX4=$(python scripts/ncu_pick.py gpurun_out/final/ncu_launches_c4.csv cgemm_f16_pair_kernel "--variant=cgemm_f16_pair_kernel<256, 1, 64, 0, 1>" --ms=7.0 --ms=9.0 --skip=1 --summary 2> gpurun_out/final/ncu_launches_c4_summary.txt); echo "idx4=$IDX4"; head -6 gpurun_out/final/ncu_launches_c4_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cgemm_f16_pair_kernel -s $IDX4 -c 1 -o gpurun_out/final/ncu_full_c4_k256 $C4 > gpurun_out/final/ncu_full_c4.log 2>&1; echo "ncu c4 rc=$?"
