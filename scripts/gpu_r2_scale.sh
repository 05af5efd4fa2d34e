# Scaling on one box: config 5 (slices) and config 4 (Bristlecone-70 slices)
# at N = 1, 2, 4 GPUs (torchrun, NCCL, checked merge), config 2 (x1 batches)
# at N = 4; the 2-GPU NCCL sliced-batch tests.
mkdir -p gpurun_out/scale
nvidia-smi --query-gpu=index,name --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -rA > gpurun_out/scale/multi_pytest.log 2>&1; echo "multi tests rc=$?"; tail -3 gpurun_out/scale/multi_pytest.log
for c in 5 4; do
  for n in 1 2 4; do
    if [ $n = 1 ]; then
      timeout 900 python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/scale/c${c}_n$n.jsonl 2> gpurun_out/scale/c${c}_n$n.err
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --config $c --steps 8 --warmup 3 > gpurun_out/scale/c${c}_n$n.jsonl 2> gpurun_out/scale/c${c}_n$n.err
    fi
    echo "c$c N=$n rc=$?: $(tail -1 gpurun_out/scale/c${c}_n$n.jsonl | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], round(d["ms_per_step"],1), "ms/step", d["config"].get("merge",{}).get("checks","")[:80])')"
  done
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29520 bench.py --gpus 4 --config 2 --steps 8 --warmup 3 > gpurun_out/scale/c2_n4.jsonl 2> gpurun_out/scale/c2_n4.err
echo "c2 N=4 rc=$?: $(tail -1 gpurun_out/scale/c2_n4.jsonl | cut -c1-150)"
