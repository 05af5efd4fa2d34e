mkdir -p gpurun_out
nvidia-smi topo -m | head -5
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2.log 2>&1; echo "n2 rc=$?"
tail -2 gpurun_out/bench_n2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 2 --warmup 1 --config 5 --no-cpu-baseline > gpurun_out/bench_n2_c5.log 2>&1; echo "n2c5 rc=$?"
tail -2 gpurun_out/bench_n2_c5.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/bench_n2_ref.log 2>&1; echo "n2ref rc=$?"
tail -1 gpurun_out/bench_n2_ref.log
