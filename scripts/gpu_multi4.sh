mkdir -p gpurun_out
for n in 1 2 4; do
if [ $n -eq 1 ]; then timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/scale_c2_n1.log 2>&1;
else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/scale_c2_n$n.log 2>&1; fi
echo "n=$n rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/scale_c2_n$n.log').read().strip().splitlines()[-1]);print(d['n_gpus'], d['value'], d['tflops_eq1'], d['ms_per_step'], d['clocks'])"
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/scale_c4_n4.log 2>&1; echo "c4 n4 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/scale_c4_n4.log').read().strip().splitlines()[-1]);print(d['n_gpus'], d['value'], d['tflops_eq1'], d['ms_per_step'], d['clocks'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/scale_ref_n2.log 2>&1; echo "ref n2 rc=$?"; tail -1 gpurun_out/scale_ref_n2.log | cut -c1-200
