mkdir -p gpurun_out/r2j
timeout 600 python tools/bench_lmhead_bwd.py 4096 32768 realistic > gpurun_out/r2j/bwd_d4096_real.json 2> gpurun_out/r2j/bwd.err
timeout 600 python tools/bench_lmhead_bwd.py 8192 16384 realistic > gpurun_out/r2j/bwd_d8192_real.json 2>> gpurun_out/r2j/bwd.err
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2j/gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r2j/gputest.log
