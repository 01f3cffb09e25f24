# K2 row claims pipelined one row deep and enabled for short rows: parity, then A/B vs HEAD
mkdir -p gpurun_out/r2aa
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vocab_parallel.py tests/test_gpu_guard.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2aa/test.log 2>&1; echo "rc=$?" >> gpurun_out/r2aa/test.log
for r in 1 2; do for v in old new; do
  if [ $v = old ]; then export ESPO_LIB=$PWD/abtmp/libespo_old.so; else unset ESPO_LIB; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --vocab-shards 8 > gpurun_out/r2aa/tp8_$v$r.json 2>/dev/null
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --vocab-shards 2 > gpurun_out/r2aa/tp2_$v$r.json 2>/dev/null
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg > gpurun_out/r2aa/c1_$v$r.json 2>/dev/null
done; done
