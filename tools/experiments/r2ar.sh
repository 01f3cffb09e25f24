# LM-head forward: lockstep chunk / slack and raster group around g16 (sustained A/B)
mkdir -p gpurun_out/r2ar
timeout 1500 python tools/bench_lmhead_fwd_ab.py 8192 2 3 sync2 > gpurun_out/r2ar/fwd_d8192.json 2> gpurun_out/r2ar/err.log
timeout 1500 python tools/bench_lmhead_fwd_ab.py 4096 3 4 sync2 > gpurun_out/r2ar/fwd_d4096.json 2>> gpurun_out/r2ar/err.log
