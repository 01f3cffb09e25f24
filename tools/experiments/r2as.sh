# LM-head GEMM core with the raster-16 + lockstep default: parity, fwd A/B, bwd sweep
mkdir -p gpurun_out/r2as
timeout 1200 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_fullsize.py tests/test_gpu_guard.py -q > gpurun_out/r2as/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2as/test.log
timeout 1200 python tools/bench_lmhead_fwd_ab.py 8192 2 3 default2 > gpurun_out/r2as/fwd_d8192.json 2> gpurun_out/r2as/err.log
timeout 1200 python tools/bench_lmhead_fwd_ab.py 4096 3 4 default2 > gpurun_out/r2as/fwd_d4096.json 2>> gpurun_out/r2as/err.log
timeout 1200 python tools/gemm_sweep.py 4096 8192 151936 3 6 > gpurun_out/r2as/sweep_d4096.json 2>> gpurun_out/r2as/err.log
timeout 1200 python tools/gemm_sweep.py 8192 8192 151936 2 4 > gpurun_out/r2as/sweep_d8192.json 2>> gpurun_out/r2as/err.log
