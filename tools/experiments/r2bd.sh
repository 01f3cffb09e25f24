# K2 larger sub-batches: C1 full width (default 16x2x6k s4 vs s12 one sub-batch vs 14x2x8k s8
# vs 16x3x4k s8) and TP8 (s8 vs s12), interleaved
mkdir -p gpurun_out/r2bd
B="python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg"
for r in 1 2; do
  for v in 0 13 14 12; do timeout 300 $B --fwd-impl $v > gpurun_out/r2bd/c1_v${v}_$r.json 2>/dev/null; done
  for v in 12 13; do timeout 300 $B --fwd-impl $v --vocab-shards 8 > gpurun_out/r2bd/tp8_v${v}_$r.json 2>/dev/null; done
done
