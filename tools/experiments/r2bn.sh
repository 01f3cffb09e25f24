# dynamic tile scheduler on by default (dz without lockstep): parity suites + A/B vs static
mkdir -p gpurun_out/r2bn
timeout 1500 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_fullsize.py tests/test_gpu_guard.py tests/test_gpu_graph.py -q > gpurun_out/r2bn/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2bn/test.log
timeout 1500 python tools/gemm_sweep.py 4096 8192 151936 3 6 dyn > gpurun_out/r2bn/bwd_d4096.json 2> gpurun_out/r2bn/err.log
timeout 1500 python tools/bench_lmhead_fwd_ab.py 4096 3 4 dyn > gpurun_out/r2bn/fwd_d4096.json 2>> gpurun_out/r2bn/err.log
timeout 1500 python tools/gemm_sweep.py 8192 8192 151936 2 4 dyn > gpurun_out/r2bn/bwd_d8192.json 2>> gpurun_out/r2bn/err.log
timeout 1500 python tools/bench_lmhead_fwd_ab.py 8192 2 3 dyn > gpurun_out/r2bn/fwd_d8192.json 2>> gpurun_out/r2bn/err.log
timeout 900 python tools/bench_lmhead_bwd.py 4096 16384 > gpurun_out/r2bn/lmbwd_dense.json 2>> gpurun_out/r2bn/err.log
timeout 900 python tools/bench_lmhead_bwd.py 4096 32768 realistic > gpurun_out/r2bn/lmbwd_real.json 2>> gpurun_out/r2bn/err.log
