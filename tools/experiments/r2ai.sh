# K2 on TP8 shard rows vs full width: instructions per source line / SASS line (where do the
# extra instructions per element at 37 KB rows go?)
mkdir -p gpurun_out/r2ai
Q="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-factored-leg --buffer-rows 8192"
$Q --vocab-shards 8 > gpurun_out/r2ai/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rowstats_tma" -s 80 -c 1 -o gpurun_out/r2ai/tp8 $Q --vocab-shards 8 > gpurun_out/r2ai/ncu1.log 2>&1
$Q > gpurun_out/r2ai/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rowstats_tma" -s 60 -c 1 -o gpurun_out/r2ai/full $Q > gpurun_out/r2ai/ncu2.log 2>&1
for r in tp8 full; do
  python tools/ncu_summary.py gpurun_out/r2ai/$r.ncu-rep > gpurun_out/r2ai/${r}_summary.txt 2>&1
  ncu -i gpurun_out/r2ai/$r.ncu-rep --page source --csv --print-source cuda > gpurun_out/r2ai/${r}_src.csv 2>&1
  ncu -i gpurun_out/r2ai/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/r2ai/${r}_sass.csv 2>&1
done
rm -f gpurun_out/r2ai/*.ncu-rep
ls -la gpurun_out/r2ai
