# Reference fixtures that need more host RAM than the build container
# (config 2: ~52 GB per slice): the unmodified reference (oracle/_ref) on
# the GPU box's host cores, written to gpurun_out/golden/.
mkdir -p gpurun_out/golden
free -g | head -2; nproc
export GOLDEN_OUT=gpurun_out/golden REF_BLAS_THREADS=$(nproc)
timeout 3000 python oracle/gen_golden_large.py config2 > gpurun_out/golden/config2.log 2>&1; echo "config2 rc=$?"; tail -3 gpurun_out/golden/config2.log
timeout 2400 python oracle/gen_golden_large.py bc70 > gpurun_out/golden/bc70.log 2>&1; echo "bc70 rc=$?"; tail -3 gpurun_out/golden/bc70.log
