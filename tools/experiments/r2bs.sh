# dW epilogue via TMA reduce-add: sustained sweep + per-launch ncu of the dW GEMM
mkdir -p gpurun_out/r2bs
timeout 1500 python tools/gemm_sweep.py 4096 8192 151936 3 6 red > gpurun_out/r2bs/red_d4096.json 2> gpurun_out/r2bs/err.log
timeout 1500 python tools/gemm_sweep.py 8192 8192 151936 2 4 red > gpurun_out/r2bs/red_d8192.json 2>> gpurun_out/r2bs/err.log
