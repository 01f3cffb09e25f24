# 256 x 512 CTA-pair GEMMs: accumulator released in halves (the next tile's first K-steps on
# columns 0-255 overlap the epilogue's read of 256-511) vs whole; parity + sustained A/B
mkdir -p gpurun_out/r2au
timeout 1200 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_fullsize.py tests/test_gpu_guard.py -q -x > gpurun_out/r2au/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2au/test.log
timeout 1200 python tools/bench_lmhead_fwd_ab.py 4096 3 4 half > gpurun_out/r2au/fwd_d4096.json 2> gpurun_out/r2au/err.log
timeout 1200 python tools/bench_lmhead_fwd_ab.py 8192 2 3 half > gpurun_out/r2au/fwd_d8192.json 2>> gpurun_out/r2au/err.log
timeout 1200 python tools/gemm_sweep.py 4096 8192 151936 3 6 half > gpurun_out/r2au/sweep_d4096.json 2>> gpurun_out/r2au/err.log
timeout 1200 python tools/gemm_sweep.py 8192 8192 151936 2 4 half > gpurun_out/r2au/sweep_d8192.json 2>> gpurun_out/r2au/err.log
