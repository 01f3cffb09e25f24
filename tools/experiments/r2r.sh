# K2 general chunks on the packed fast path (finite −1e30 patching): parity, then A/B vs the
# previous library on the TP8 shard rows and at full width (ESPO_LIB = old build)
mkdir -p gpurun_out/r2r
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_vocab_parallel.py tests/test_gpu_guard.py -x -q > gpurun_out/r2r/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2r/test.log
for r in 1 2; do for v in old new; do
  if [ $v = old ]; then export ESPO_LIB=$PWD/abtmp/libespo_old.so; else unset ESPO_LIB; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --vocab-shards 8 > gpurun_out/r2r/tp8_$v$r.json 2>/dev/null
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg > gpurun_out/r2r/c1_$v$r.json 2>/dev/null
done; done
