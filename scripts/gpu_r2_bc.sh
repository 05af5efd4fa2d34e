# Bristlecone-60/70 bench lines with per-op profiles, then the k=256 profile.
mkdir -p gpurun_out
timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/r2_ops_c4.jsonl > gpurun_out/r2_bench_c4.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/r2_bench_c4.log | cut -c1-300
timeout 900 python bench.py --config 3 --steps 8 --warmup 3 --no-cpu-baseline --profile-out gpurun_out/r2_ops_c3.jsonl > gpurun_out/r2_bench_c3.log 2>&1; echo "c3 rc=$?"; tail -1 gpurun_out/r2_bench_c3.log | cut -c1-300
bash scripts/gpu_r2_prof_k256.sh
