# LM-head forward: GEMM soft lockstep and raster groups, sustained A/B (d = 8192, 4096)
mkdir -p gpurun_out/r2aq
timeout 1200 python tools/bench_lmhead_fwd_ab.py 8192 2 3 sync > gpurun_out/r2aq/fwd_d8192.json 2> gpurun_out/r2aq/err.log
timeout 1200 python tools/bench_lmhead_fwd_ab.py 4096 3 4 sync > gpurun_out/r2aq/fwd_d4096.json 2>> gpurun_out/r2aq/err.log
