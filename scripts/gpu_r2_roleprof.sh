# Pair-kernel role timelines (QSG_TC_PROF=1: per-CTA wait / busy cycles per
# launch, diagnostics only) on configs 4 and 2; kernel tests first.
mkdir -p gpurun_out/rp
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider > gpurun_out/rp/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/rp/pytest.log
for c in 4 2; do
  QSG_TC_PROF=1 timeout 900 python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/rp/c$c.log 2> gpurun_out/rp/c$c.err; echo "c$c rc=$?"
  grep qsg-prof gpurun_out/rp/c$c.err | sort | uniq -c | sort -rn | head -12
done
