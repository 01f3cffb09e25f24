# GEMM-core barrier waits without .acquire.cluster (no L1 invalidation per poll): parity and
# A/B against the previous build (ESPO_LIB=ab/libespo_prev.so), alternating processes
mkdir -p gpurun_out/r2bb
timeout 1200 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_fullsize.py tests/test_gpu_guard.py tests/test_gpu_graph.py -q -x > gpurun_out/r2bb/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2bb/test.log
for r in 1 2; do
  timeout 900 python tools/bench_lmhead_fwd_ab.py 4096 2 4 default2 > gpurun_out/r2bb/fwd4096_new_$r.json 2>/dev/null
  ESPO_LIB=ab/libespo_prev.so timeout 900 python tools/bench_lmhead_fwd_ab.py 4096 2 4 default2 > gpurun_out/r2bb/fwd4096_prev_$r.json 2>/dev/null
  timeout 900 python tools/gemm_sweep.py 4096 8192 151936 2 6 > gpurun_out/r2bb/bwd4096_new_$r.json 2>/dev/null
  ESPO_LIB=ab/libespo_prev.so timeout 900 python tools/gemm_sweep.py 4096 8192 151936 2 6 > gpurun_out/r2bb/bwd4096_prev_$r.json 2>/dev/null
done
timeout 900 python tools/bench_lmhead_fwd_ab.py 8192 2 3 default2 > gpurun_out/r2bb/fwd8192_new.json 2>/dev/null
ESPO_LIB=ab/libespo_prev.so timeout 900 python tools/bench_lmhead_fwd_ab.py 8192 2 3 default2 > gpurun_out/r2bb/fwd8192_prev.json 2>/dev/null
