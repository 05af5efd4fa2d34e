# Bristlecone-70 reference fixture for two contributing slices (2, 6), on the GPU box host.
mkdir -p gpurun_out/golden
export GOLDEN_OUT=gpurun_out/golden REF_BLAS_THREADS=$(nproc)
timeout 2400 python oracle/gen_golden_large.py bc70 > gpurun_out/golden/bc70.log 2>&1; echo "bc70 rc=$?"; tail -3 gpurun_out/golden/bc70.log
