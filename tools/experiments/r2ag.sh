mkdir -p gpurun_out/r2ag
for impl in 0 2 3 4 5 7; do
  timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --vocab-shards 8 --fwd-impl $impl > gpurun_out/r2ag/tp8_$impl.json 2>/dev/null
done
