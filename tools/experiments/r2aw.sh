# K2 per-chunk bookkeeping on 32-bit shared addresses + incremental source pointer: parity and
# interleaved A/B against the previous build (ab/libespo_prev.so via ESPO_LIB)
mkdir -p gpurun_out/r2aw
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vocab_parallel.py tests/test_gpu_edges.py tests/test_gpu_guard.py tests/test_gpu_bench_emulate.py tests/test_gpu_fullsize.py -q > gpurun_out/r2aw/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2aw/test.log
B="python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg"
for round in 1 2; do
  timeout 300 $B > gpurun_out/r2aw/c1_new_$round.json 2>/dev/null
  ESPO_LIB=ab/libespo_prev.so timeout 300 $B > gpurun_out/r2aw/c1_prev_$round.json 2>/dev/null
  timeout 300 $B --vocab-shards 8 > gpurun_out/r2aw/tp8_new_$round.json 2>/dev/null
  ESPO_LIB=ab/libespo_prev.so timeout 300 $B --vocab-shards 8 > gpurun_out/r2aw/tp8_prev_$round.json 2>/dev/null
done
