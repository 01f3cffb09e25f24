# dh / dW lockstep on by default above d = 4096 (dh groups of 16): parity + sweeps
mkdir -p gpurun_out/r2az
timeout 1200 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_fullsize.py tests/test_gpu_guard.py -q -x > gpurun_out/r2az/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2az/test.log
timeout 1500 python tools/gemm_sweep.py 8192 8192 151936 3 4 sync > gpurun_out/r2az/sweep_d8192.json 2> gpurun_out/r2az/err.log
timeout 1500 python tools/gemm_sweep.py 4096 8192 151936 3 6 > gpurun_out/r2az/sweep_d4096.json 2>> gpurun_out/r2az/err.log
