# dynamic tile scheduler: LM-head forward and backward A/B (sustained, interleaved; fair cuBLAS leg)
mkdir -p gpurun_out/r2bm
timeout 1500 python tools/gemm_sweep.py 4096 8192 151936 3 6 dyn > gpurun_out/r2bm/bwd_d4096.json 2> gpurun_out/r2bm/err.log
timeout 1500 python tools/bench_lmhead_fwd_ab.py 4096 3 4 dyn > gpurun_out/r2bm/fwd_d4096.json 2>> gpurun_out/r2bm/err.log
timeout 1500 python tools/gemm_sweep.py 8192 8192 151936 2 4 dyn > gpurun_out/r2bm/bwd_d8192.json 2>> gpurun_out/r2bm/err.log
timeout 1500 python tools/bench_lmhead_fwd_ab.py 8192 2 3 dyn > gpurun_out/r2bm/fwd_d8192.json 2>> gpurun_out/r2bm/err.log
