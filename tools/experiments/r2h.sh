mkdir -p gpurun_out/r2h
timeout 900 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_fullsize.py tests/test_gpu_guard.py -x -q > gpurun_out/r2h/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2h/test.log
timeout 600 python tools/bench_lmhead_bwd.py 4096 16384 > gpurun_out/r2h/bwd_d4096.json 2> gpurun_out/r2h/bwd_d4096.err
