# Config 3: per-step device time vs the sum of its kernels (GPU idle between
# launches of one eager slice), one step under an ncu launch list.
mkdir -p gpurun_out/gap
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/gap/bench_c3.log 2>&1; tail -1 gpurun_out/gap/bench_c3.log | cut -c1-200
QSG_GRAPH=0 timeout 600 python bench.py --config 2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/gap/bench_c2_nograph.log 2>&1; tail -1 gpurun_out/gap/bench_c2_nograph.log | cut -c1-200
timeout 600 python bench.py --config 2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/gap/bench_c2.log 2>&1; tail -1 gpurun_out/gap/bench_c2.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gap/launches_c3.csv python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
