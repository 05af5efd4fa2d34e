# Round-end refresh: GPU tests, smoke, the default bench line (with the CPU
# baseline), the reference arm, and config 1 (batched) with its e2e.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/re_pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/re_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/re_smoke.log
timeout 900 python bench.py > gpurun_out/re_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/re_bench.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/re_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/re_ref.log | cut -c1-300
timeout 600 python bench.py --config 1 > gpurun_out/re_bench_c1.log 2>&1; echo "c1 rc=$?"; tail -1 gpurun_out/re_bench_c1.log | cut -c1-300
