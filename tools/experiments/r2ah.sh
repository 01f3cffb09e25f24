mkdir -p gpurun_out/r2ah
timeout 900 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_fullsize.py tests/test_gpu_guard.py -q > gpurun_out/r2ah/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2ah/test.log
timeout 900 python tools/gemm_sweep.py 4096 8192 151936 3 6 > gpurun_out/r2ah/sweep_d4096.json 2>> gpurun_out/r2ah/err.log
timeout 900 python tools/gemm_sweep.py 4096 6000 151936 3 6 > gpurun_out/r2ah/sweep_d4096_n6000.json 2>> gpurun_out/r2ah/err.log
timeout 900 python tools/gemm_sweep.py 8192 8192 151936 2 4 > gpurun_out/r2ah/sweep_d8192.json 2>> gpurun_out/r2ah/err.log
