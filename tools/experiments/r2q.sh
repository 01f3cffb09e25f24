mkdir -p gpurun_out/r2q
timeout 900 python tools/bench_lmhead_bwd.py 4096 32768 realistic > gpurun_out/r2q/bwd_d4096_real.json 2> gpurun_out/r2q/bwd.err
timeout 900 python tools/bench_lmhead_bwd.py 4096 16384 > gpurun_out/r2q/bwd_d4096_dense.json 2>> gpurun_out/r2q/bwd.err
