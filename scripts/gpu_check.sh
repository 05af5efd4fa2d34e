mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2; lscpu | grep "Model name"
python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench1.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/bench1.log
