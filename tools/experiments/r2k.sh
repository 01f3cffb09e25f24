mkdir -p gpurun_out/r2k
timeout 900 python tools/gemm_sweep.py 4096 8192 151936 3 6 > gpurun_out/r2k/sweep_d4096_burst6.json 2> gpurun_out/r2k/err.log
timeout 900 python tools/gemm_sweep.py 4096 8192 151936 5 1 > gpurun_out/r2k/sweep_d4096_burst1.json 2>> gpurun_out/r2k/err.log
