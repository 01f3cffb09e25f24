# LM-head backward: soft lockstep on the dh / dW GEMMs (sustained sweep, d = 8192 and 4096)
mkdir -p gpurun_out/r2at
timeout 1500 python tools/gemm_sweep.py 8192 8192 151936 2 4 sync > gpurun_out/r2at/sweep_d8192.json 2> gpurun_out/r2at/err.log
timeout 1500 python tools/gemm_sweep.py 4096 8192 151936 3 6 sync > gpurun_out/r2at/sweep_d4096.json 2>> gpurun_out/r2at/err.log
