# LM-head backward vs cuBLAS GEMMs on the SAME recompute and compaction (fixed sweep leg);
# dW raster / L2 policy / tile-width variants (dense 8192-row sub-chunks, sustained)
mkdir -p gpurun_out/r2bf
timeout 1500 python tools/gemm_sweep.py 4096 8192 151936 3 6 dwr > gpurun_out/r2bf/dwr_d4096.json 2> gpurun_out/r2bf/err.log
timeout 1500 python tools/gemm_sweep.py 8192 8192 151936 2 4 > gpurun_out/r2bf/def_d8192.json 2>> gpurun_out/r2bf/err.log
