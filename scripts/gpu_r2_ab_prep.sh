# 3M prep kernels vectorised: kernel + engine + full-size parity tests, then
# same-box A/B against the previous build on configs 2 and 5, and a launch list of config 2.
mkdir -p gpurun_out/abp
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_large.py -m gpu -q -x -p no:cacheprovider > gpurun_out/abp/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/abp/pytest.log
for r in 1 2; do
  for v in "QSG_LIB=$PWD/ab/libqsg_base.so" "QSG_LIB=$PWD/paper_1905_00444_b200/libqsg.so"; do
    tag=$(basename ${v#QSG_LIB=} .so)
    for c in 2 5; do
      env $v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/abp/bench_c${c}_${tag}_$r.log 2>&1
      echo "$tag run $r c$c: $(tail -1 gpurun_out/abp/bench_c${c}_${tag}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), "ms/step", d["clocks"]["sm_mhz"], "MHz")')"
    done
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:tc3m_prep --log-file gpurun_out/abp/prep_launches.csv python bench.py --config 2 --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
