mkdir -p gpurun_out/r2v
timeout 900 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_fullsize.py tests/test_gpu_guard.py -q > gpurun_out/r2v/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2v/test.log
timeout 900 python tools/bench_lmhead_fwd_ab.py 4096 3 4 > gpurun_out/r2v/fwd_d4096.json 2> gpurun_out/r2v/err.log
timeout 900 python tools/bench_lmhead_fwd_ab.py 8192 2 3 > gpurun_out/r2v/fwd_d8192.json 2>> gpurun_out/r2v/err.log
timeout 900 python tools/gemm_sweep.py 4096 8192 151936 3 6 > gpurun_out/r2v/sweep_d4096.json 2>> gpurun_out/r2v/err.log
