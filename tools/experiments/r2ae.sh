mkdir -p gpurun_out/r2ae
timeout 900 python tools/bench_lmhead_fwd_ab.py 4096 3 4 > gpurun_out/r2ae/fwd_d4096.json 2> gpurun_out/r2ae/err.log
timeout 900 python tools/bench_lmhead_fwd_ab.py 8192 2 3 > gpurun_out/r2ae/fwd_d8192.json 2>> gpurun_out/r2ae/err.log
timeout 900 python tools/gemm_sweep.py 4096 8192 151936 3 6 > gpurun_out/r2ae/sweep_d4096.json 2>> gpurun_out/r2ae/err.log
timeout 900 python tools/gemm_sweep.py 8192 8192 151936 2 4 > gpurun_out/r2ae/sweep_d8192.json 2>> gpurun_out/r2ae/err.log
