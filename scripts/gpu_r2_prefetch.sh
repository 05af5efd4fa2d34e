# L2 prefetch of pre-split A boxes k-blocks ahead (QSG_TC_PREFETCH=P) on the
# latency-bound k = 256 class: role counters + speed on configs 4, 3, 2.
mkdir -p gpurun_out/pf
timeout 600 python -m pytest tests/test_gpu_engine.py -m gpu -q -x -p no:cacheprovider -k "split or config2" > gpurun_out/pf/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pf/pytest.log
for P in 4 8 16; do
  QSG_TC_PREFETCH=$P QSG_TC_PROF=1 timeout 900 python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2> gpurun_out/pf/prof_c4_P$P.err
  echo "P=$P $(grep qsg-prof gpurun_out/pf/prof_c4_P$P.err | grep 'm=8388608 n=256 k=256' | head -1)"
done
for r in 1 2; do
  for P in 0 4 8 16; do
    for c in 4 3 2; do
      QSG_TC_PREFETCH=$P python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/pf/bench_c${c}_P${P}_$r.log 2>&1
      echo "P=$P run $r c$c: $(tail -1 gpurun_out/pf/bench_c${c}_P${P}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")')"
    done
  done
done
