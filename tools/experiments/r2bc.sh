# K2 at 1/8-vocabulary shard rows: one 8-vector sub-batch per 4 KB chunk (variant 12) vs the
# default two 4-vector sub-batches; interleaved bench A/B + parity of the variant
mkdir -p gpurun_out/r2bc
B="python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --vocab-shards 8"
for r in 1 2 3; do
  timeout 300 $B > gpurun_out/r2bc/tp8_def_$r.json 2>/dev/null
  timeout 300 $B --fwd-impl 12 > gpurun_out/r2bc/tp8_v12_$r.json 2>/dev/null
done
timeout 300 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --vocab-shards 4 > gpurun_out/r2bc/tp4_def.json 2>/dev/null
timeout 300 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --vocab-shards 4 --fwd-impl 12 > gpurun_out/r2bc/tp4_v12.json 2>/dev/null
