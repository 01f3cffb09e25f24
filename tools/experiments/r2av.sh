# LM-head backward: dW on 512-wide pair tiles now that the accumulator is released in halves
mkdir -p gpurun_out/r2av
timeout 1500 python tools/gemm_sweep.py 4096 8192 151936 3 6 dw > gpurun_out/r2av/sweep_d4096.json 2> gpurun_out/r2av/err.log
timeout 1500 python tools/gemm_sweep.py 8192 8192 151936 2 4 dw > gpurun_out/r2av/sweep_d8192.json 2>> gpurun_out/r2av/err.log
