mkdir -p gpurun_out/r2p
timeout 900 python -m pytest tests/test_gpu_lmhead.py -x -q > gpurun_out/r2p/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2p/test.log
timeout 900 python tools/gemm_sweep.py 4096 8192 151936 3 6 > gpurun_out/r2p/sweep_d4096_burst6.json 2> gpurun_out/r2p/err.log
timeout 900 python tools/gemm_sweep.py 8192 8192 151936 2 4 > gpurun_out/r2p/sweep_d8192_burst4.json 2>> gpurun_out/r2p/err.log
