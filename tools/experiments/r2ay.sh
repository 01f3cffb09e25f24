# dh / dW soft lockstep with chunks counted from each item's first K-step (split-K halves no
# longer wait on counts their wave never reaches); LM-head parity; sustained sweeps
mkdir -p gpurun_out/r2ay
timeout 1200 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_fullsize.py -q -x > gpurun_out/r2ay/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2ay/test.log
timeout 1500 python tools/gemm_sweep.py 4096 8192 151936 3 6 sync > gpurun_out/r2ay/sweep_d4096.json 2> gpurun_out/r2ay/err.log
timeout 1500 python tools/gemm_sweep.py 8192 8192 151936 2 4 sync > gpurun_out/r2ay/sweep_d8192.json 2>> gpurun_out/r2ay/err.log
