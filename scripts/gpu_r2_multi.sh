# 2-GPU box: NCCL sliced-batch tests, full-size fp64 parity, torchrun bench
# (config 5, checked merge), Bristlecone-60/70 bench lines.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name,clocks.sm,power.draw --format=csv,noheader
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_large.py -m gpu -q -p no:cacheprovider -rA > gpurun_out/r2_multi_pytest.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2_multi_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 4 --warmup 3 > gpurun_out/r2_bench_c5_n2.log 2> gpurun_out/r2_bench_c5_n2.err; echo "c5 n2 rc=$?"; tail -1 gpurun_out/r2_bench_c5_n2.log | cut -c1-300
timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline --profile-out gpurun_out/r2_ops_c4.jsonl > gpurun_out/r2_bench_c4.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/r2_bench_c4.log | cut -c1-400
timeout 900 python bench.py --config 3 --steps 8 --warmup 3 --no-cpu-baseline --profile-out gpurun_out/r2_ops_c3.jsonl > gpurun_out/r2_bench_c3.log 2>&1; echo "c3 rc=$?"; tail -1 gpurun_out/r2_bench_c3.log | cut -c1-400
