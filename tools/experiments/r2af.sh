mkdir -p gpurun_out/r2af
ESPO_DEBUG=1 timeout 300 python tools/lmhead_bwd_once.py 4096 8192 0 > gpurun_out/r2af/once.log 2>&1
ESPO_DEBUG=1 timeout 300 python tools/lmhead_bwd_once.py 4096 8192 5 >> gpurun_out/r2af/once.log 2>&1
timeout 900 python tools/bench_lmhead_fwd_ab.py 4096 3 4 > gpurun_out/r2af/fwd_d4096.json 2> gpurun_out/r2af/err.log
timeout 900 python tools/gemm_sweep.py 4096 8192 151936 3 6 > gpurun_out/r2af/sweep_d4096.json 2>> gpurun_out/r2af/err.log
