# LM-head backward on the tcgen05 GEMMs: parity tests, then the d=4096 benchmark
mkdir -p gpurun_out/r2b
timeout 900 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_fullsize.py -x -q > gpurun_out/r2b/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2b/test.log
timeout 600 python tools/bench_lmhead_bwd.py 4096 16384 > gpurun_out/r2b/bwd_d4096.json 2> gpurun_out/r2b/bwd_d4096.err
