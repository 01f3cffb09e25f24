# chunk size of the bench's two-sweep pass: 32,768 vs 65,536 rows per call (per-call gaps)
mkdir -p gpurun_out/r2be
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg"
for r in 1 2 3; do
  timeout 300 $B > gpurun_out/r2be/c32k_$r.json 2>/dev/null
  timeout 300 $B --buffer-rows 65536 > gpurun_out/r2be/c64k_$r.json 2>/dev/null
done
