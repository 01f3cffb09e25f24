# bench-level A/B of K2 ring geometries, interleaved: C1 (full width) and TP8 / TP4 shard rows
mkdir -p gpurun_out/r2an
B="python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg"
for round in 1 2; do
  for impl in 0 16 18; do
    timeout 300 $B --fwd-impl $impl > gpurun_out/r2an/c1_${impl}_$round.json 2>/dev/null
    timeout 300 $B --fwd-impl $impl --vocab-shards 8 > gpurun_out/r2an/tp8_${impl}_$round.json 2>/dev/null
  done
  for impl in 0 16 17; do
    timeout 300 $B --fwd-impl $impl --vocab-shards 4 > gpurun_out/r2an/tp4_${impl}_$round.json 2>/dev/null
  done
done
